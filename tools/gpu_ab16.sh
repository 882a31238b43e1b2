#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/a_build.log 2>&1
B="python bench.py --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --no-schedule --phases"
timeout 900 $B --steps 10 > gpurun_out/c_c3.json 2> gpurun_out/c_c3.err
timeout 600 $B --config C2 --steps 20 > gpurun_out/c_c2.json 2> gpurun_out/c_c2.err
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "hvp or pcg_matches or chunked or trajectory or batch_equals or streamed or c2_contact" > gpurun_out/c_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/c_tests.log
