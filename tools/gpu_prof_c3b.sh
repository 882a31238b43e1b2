#!/bin/bash
# ncu --set full of the streamed k_pcg and k_assemble_soft on C3 (first launches of step 3), raw + source pages
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/p_build.log 2>&1
L="--no-e2e --no-schedule --no-cpu-baseline --no-alongside"
for K in k_pcg k_assemble_soft; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^${K}$" --launch-skip 0 --launch-count 1 -o /tmp/p_${K}_c3 -f python bench.py --config C3 --steps 1 --warmup 3 $L > gpurun_out/p_ncu_${K}_c3.log 2>&1
  ncu -i /tmp/p_${K}_c3.ncu-rep --page raw --csv > gpurun_out/p_${K}_c3_raw.csv 2>/dev/null
  ncu -i /tmp/p_${K}_c3.ncu-rep --page source --csv > gpurun_out/p_${K}_c3_source.csv 2>/dev/null
  ncu -i /tmp/p_${K}_c3.ncu-rep --page details --csv > gpurun_out/p_${K}_c3_details.csv 2>/dev/null
done
timeout 600 python tools/diag_c5.py 128 80 > gpurun_out/d_c5.log 2>&1
