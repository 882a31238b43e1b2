#!/bin/bash
# experiments: streamed-PCG ELL parity + C3/C2 lockstep with lm_mu0 10 vs 1
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/q_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "streamed or pcg_matches" > gpurun_out/q_ell_tests.log 2>&1
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --phases"
timeout 900 $B --config C3 > gpurun_out/q_c3_ell.json 2> gpurun_out/q_c3_ell.err
timeout 900 $B --config C3 --set lm_mu0=1.0 > gpurun_out/q_c3_mu1.json 2> gpurun_out/q_c3_mu1.err
timeout 600 $B --config C2 --steps 20 > gpurun_out/q_c2_mu10.json 2> gpurun_out/q_c2_mu10.err
timeout 600 $B --config C2 --steps 20 --set lm_mu0=1.0 > gpurun_out/q_c2_mu1.json 2> gpurun_out/q_c2_mu1.err
