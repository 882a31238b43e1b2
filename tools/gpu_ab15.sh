#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/a_build.log 2>&1
timeout 1800 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_contact.py tests/test_gpu_fullsize.py -k "not c5 and not c4 and not cluster and not relaxed" > gpurun_out/a_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/a_tests.log
