#!/bin/bash
# streamed-PCG changes: parity on the streamed path + C3 bench A/B (2 vs 3 CTAs/SM)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/a_build.log 2>&1
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_fullsize.py tests/test_gpu_parity.py -k "c3 or streamed or chunked or hvp" > gpurun_out/a_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/a_tests.log
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --no-schedule --phases"
timeout 900 $B > gpurun_out/a_c3.json 2> gpurun_out/a_c3.err

