#!/bin/bash
# full GPU tests + default bench + relaxed-tolerance (R22) bench variants
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/gpu_r2.sh
B="python bench.py --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --no-schedule"
timeout 900 $B --config C3 --steps 10 --set pcg_eta_max=0.1 > gpurun_out/e_c3_ew.json 2> gpurun_out/e_c3_ew.err
timeout 600 $B --config C2 --steps 20 --set pcg_eta_max=0.1 > gpurun_out/e_c2_ew.json 2> gpurun_out/e_c2_ew.err
timeout 600 $B --config C2 --steps 20 > gpurun_out/e_c2.json 2> gpurun_out/e_c2.err
