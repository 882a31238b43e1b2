#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/h_build.log 2>&1
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_grasp.py tests/test_gpu_contact.py tests/test_gpu_fullsize.py -k "c4 or c5 or cluster or relaxed" > gpurun_out/h_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/h_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/h_smoke.log
timeout 1500 python bench.py --phases > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
