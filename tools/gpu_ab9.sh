#!/bin/bash
# streaming cache hints on the operator + compacted residual Hessians: parity subset, C3/C2 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/a_build.log 2>&1
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_fullsize.py tests/test_gpu_contact.py tests/test_gpu_parity.py -k "c3_after or soft_soft or streamed or pcg_matches or capacity or lm_exact or hvp or chunked" > gpurun_out/a_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/a_tests.log
B="python bench.py --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --no-schedule --phases"
timeout 900 $B --steps 10 > gpurun_out/a_c3.json 2> gpurun_out/a_c3.err
timeout 600 $B --config C2 --steps 20 > gpurun_out/a_c2.json 2> gpurun_out/a_c2.err
L="--no-e2e --no-schedule --no-cpu-baseline --no-alongside"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_pcg" --launch-skip 0 --launch-count 1 -o /tmp/f_k_pcg_C3 -f python bench.py --config C3 --envs-total 1024 --steps 1 --warmup 3 $L > gpurun_out/f_ncu_k_pcg_C3.log 2>&1
ncu -i /tmp/f_k_pcg_C3.ncu-rep --page raw --csv > gpurun_out/f_k_pcg_C3_raw.csv 2>/dev/null
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
timeout 900 ncu --profile-from-start off -k regex:"^k_pcg" $M --csv --log-file gpurun_out/f_traffic_c3.csv python tools/pcg_traffic.py C3 4096 5 > gpurun_out/f_traffic_c3.log 2>&1
