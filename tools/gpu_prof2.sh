#!/bin/bash
# k_pcg per-section clocks (instrumented build, C3), PCG DRAM traffic per launch (C3, C2) for bench's
# roofline.traffic, ncu --set full of k_tets / k_pairs_x / k_linesearch on C3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/q_build.log 2>&1
bash tools/build_clocks.sh > gpurun_out/q_build_clk.log 2>&1
timeout 600 python tools/pcg_clocks.py 4096 3 2 C3 > gpurun_out/q_clocks_c3.log 2>&1
rm -f paper_2504_12908_b200/libtaccel_cuda_clk.so
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
timeout 900 ncu --profile-from-start off -k regex:"^k_pcg" $M --csv --log-file gpurun_out/q_traffic_c3.csv python tools/pcg_traffic.py C3 4096 5 > gpurun_out/q_traffic_c3.log 2>&1
timeout 600 ncu --profile-from-start off -k regex:"^k_pcg" $M --csv --log-file gpurun_out/q_traffic_c2.csv python tools/pcg_traffic.py C2 1024 12 > gpurun_out/q_traffic_c2.log 2>&1
L="--no-e2e --no-schedule --no-cpu-baseline --no-alongside"
for K in k_tets k_pairs_x k_linesearch; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${K}$" --launch-skip 0 --launch-count 1 -o /tmp/q_${K}_c3 -f python bench.py --config C3 --steps 1 --warmup 3 $L > gpurun_out/q_ncu_${K}_c3.log 2>&1
  ncu -i /tmp/q_${K}_c3.ncu-rep --page raw --csv > gpurun_out/q_${K}_c3_raw.csv 2>/dev/null
  ncu -i /tmp/q_${K}_c3.ncu-rep --page source --csv > gpurun_out/q_${K}_c3_source.csv 2>/dev/null
done
