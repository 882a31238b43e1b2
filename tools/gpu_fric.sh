#!/bin/bash
# friction vs frictionless peg workloads (Newton tails), C5 with the corrected hand geometry
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/f_build.log 2>&1
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --no-schedule"
timeout 900 $B --config C3 --set mu_friction=0.5 > gpurun_out/f_c3_mu05.json 2> gpurun_out/f_c3_mu05.err
timeout 600 $B --config C2 --steps 20 --set mu_friction=0.5 > gpurun_out/f_c2_mu05.json 2> gpurun_out/f_c2_mu05.err
timeout 600 $B --config C2 --steps 20 --warmup 30 --set mu_friction=0.5 > gpurun_out/f_c2_mu05_w30.json 2> gpurun_out/f_c2_mu05_w30.err
timeout 600 $B --config C2 --steps 20 --warmup 30 > gpurun_out/f_c2_w30.json 2> gpurun_out/f_c2_w30.err
timeout 600 python tools/diag_c5.py 128 80 > gpurun_out/f_c5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_grasp.py -m gpu -q -x > gpurun_out/f_grasp.log 2>&1
