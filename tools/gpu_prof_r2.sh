#!/bin/bash
# per-iteration tail profile (C2, C3) and ncu --set full of the streamed k_pcg (C3, full-grid launches)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/q_build.log 2>&1
timeout 600 python tools/dbg_r2.py iters C2 > gpurun_out/q_iters_c2.log 2>&1
B="python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-schedule --no-cpu-baseline --no-alongside"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pcg\b|k_pcg\(" --launch-skip 0 --launch-count 2 -o /tmp/q_pcg_c3 -f $B > gpurun_out/q_ncu_c3.log 2>&1
ncu -i /tmp/q_pcg_c3.ncu-rep --page raw --csv > gpurun_out/q_pcg_c3_raw.csv 2>/dev/null
ncu -i /tmp/q_pcg_c3.ncu-rep --page source --csv > gpurun_out/q_pcg_c3_source.csv 2>/dev/null
