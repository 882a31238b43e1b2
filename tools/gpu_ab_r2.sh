#!/bin/bash
# round-2 A/B + profile: tests, C2 bench with the cluster PCG vs the round-1 resident PCG, ncu of k_pcg_cl
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/q_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contact.py -m gpu -q -rA > gpurun_out/q_tests.log 2>&1
B="python bench.py --config C2 --steps 10 --no-e2e --no-cpu-baseline --phases"
timeout 400 $B > gpurun_out/q_c2_cl.json 2> gpurun_out/q_c2_cl.err
TAC_PCG_CLUSTER=0 timeout 400 $B > gpurun_out/q_c2_r.json 2> gpurun_out/q_c2_r.err
TAC_COMPACT=0 timeout 400 $B > gpurun_out/q_c2_nocompact.json 2> gpurun_out/q_c2_nocompact.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_cl --launch-skip 40 --launch-count 1 -o gpurun_out/q_pcgcl -f python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-schedule --no-cpu-baseline > gpurun_out/q_ncu.log 2>&1
