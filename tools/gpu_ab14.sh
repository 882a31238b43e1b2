#!/bin/bash
# k_linesearch / k_narrow at a 3-CTA/SM budget; larger dt on C3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/a_build.log 2>&1
B="python bench.py --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --no-schedule --phases"
timeout 900 $B --steps 10 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
TAC_LS_MINB=3 TAC_NARROW_MINB=3 timeout 900 $B --steps 10 > gpurun_out/b_c3_m3.json 2> gpurun_out/b_c3_m3.err
timeout 600 $B --config C2 --steps 20 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
TAC_LS_MINB=3 TAC_NARROW_MINB=3 timeout 600 $B --config C2 --steps 20 > gpurun_out/b_c2_m3.json 2> gpurun_out/b_c2_m3.err
timeout 900 $B --steps 10 --set dt=0.04 > gpurun_out/b_c3_dt04.json 2> gpurun_out/b_c3_dt04.err
