#!/bin/bash
# k_asm_edges + k_tets_x + PCG outlining: parity subset, C3/C2 bench, C3 with the 3-CTA/SM k_pcg
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/a_build.log 2>&1
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_fullsize.py tests/test_gpu_parity.py -k "c3_after or c2_contact or streamed or chunked or hvp or trajectory or batch_equals or pcg_matches" > gpurun_out/a_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/a_tests.log
B="python bench.py --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --no-schedule --phases"
timeout 900 $B --steps 10 > gpurun_out/a_c3.json 2> gpurun_out/a_c3.err
timeout 600 $B --config C2 --steps 20 > gpurun_out/a_c2.json 2> gpurun_out/a_c2.err
TAC_PCG_STREAM_MINB=3 timeout 900 $B --steps 10 > gpurun_out/a_c3_m3.json 2> gpurun_out/a_c3_m3.err
