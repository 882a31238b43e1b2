#!/bin/bash
# checkpoint: C3 bench (streamed PCG, d in smem), C3 failure diagnostics, all GPU tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/q_build.log 2>&1
timeout 900 python bench.py --config C3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --phases > gpurun_out/q_c3_dsm.json 2> gpurun_out/q_c3_dsm.err
timeout 1500 python tools/dbg_r2.py c3 > gpurun_out/q_c3_fail.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=30 > gpurun_out/r2c_gputest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2c_gputest.log
