#!/bin/bash
# round-2 GPU check: build, GPU tests (all, with durations), default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/r2_build.log 2>&1
timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q -rA --durations=40 ${PYTEST_ARGS} > gpurun_out/r2_gputest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gputest.log
if [ -z "$NO_BENCH" ]; then
  timeout 1200 python bench.py --phases ${BENCH_ARGS} > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
  echo "bench exit $?" >> gpurun_out/r2_bench.err
fi
