#!/bin/bash
# final re-check at the last commit: GPU suite, smoke, default bench line, C4/C5 lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/g_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=30 > gpurun_out/g_gputest.log 2>&1
echo "pytest exit $?" >> gpurun_out/g_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/g_smoke.log
timeout 1500 python bench.py --phases > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
timeout 900 python bench.py --config C4 --phases --no-cpu-baseline > gpurun_out/g_bench_c4.json 2> gpurun_out/g_bench_c4.err
timeout 900 python bench.py --config C5 --phases --no-cpu-baseline > gpurun_out/g_bench_c5.json 2> gpurun_out/g_bench_c5.err
