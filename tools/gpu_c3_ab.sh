#!/bin/bash
# C3 A/B: cluster PCG (default) vs the streamed k_pcg, short lockstep bench; C3 failing-env diagnostics
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/q_build.log 2>&1
B="python bench.py --config C3 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --phases"
timeout 900 $B > gpurun_out/q_c3_cl.json 2> gpurun_out/q_c3_cl.err
TAC_PCG_CLUSTER=0 timeout 900 $B > gpurun_out/q_c3_stream.json 2> gpurun_out/q_c3_stream.err
timeout 1200 python tools/dbg_r2.py c3 > gpurun_out/q_c3_fail.log 2>&1
