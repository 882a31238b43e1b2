#!/bin/bash
# tail-split PCG A/B on C2 and C3 lockstep (TAC_PCG_TAIL_NEWTON 0 / 12), C3 iteration profile
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/q_build.log 2>&1
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --phases"
timeout 900 $B --config C3 > gpurun_out/q_tail0_c3.json 2> gpurun_out/q_tail0_c3.err
TAC_PCG_TAIL_NEWTON=12 timeout 900 $B --config C3 > gpurun_out/q_tail12_c3.json 2> gpurun_out/q_tail12_c3.err
timeout 600 $B --config C2 --steps 20 > gpurun_out/q_tail0_c2.json 2> gpurun_out/q_tail0_c2.err
TAC_PCG_TAIL_NEWTON=12 timeout 600 $B --config C2 --steps 20 > gpurun_out/q_tail12_c2.json 2> gpurun_out/q_tail12_c2.err
TAC_PCG_TAIL_NEWTON=12 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "trajectory or batch_equals or schedule" > gpurun_out/q_tail_tests.log 2>&1
