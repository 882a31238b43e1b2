#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/z_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=20 > gpurun_out/z_gputest.log 2>&1
echo "pytest exit $?" >> gpurun_out/z_gputest.log
