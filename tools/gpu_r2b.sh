#!/bin/bash
# round-2 checkpoint: build, all GPU tests, default bench (C3 + C2 alongside, no CPU baseline)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/r2b_build.log 2>&1
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -rA --durations=40 ${PYTEST_ARGS} > gpurun_out/r2b_gputest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2b_gputest.log
timeout 1500 python bench.py --phases --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
echo "bench exit $?" >> gpurun_out/r2b_bench.err
