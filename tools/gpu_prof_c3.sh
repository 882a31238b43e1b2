#!/bin/bash
# ncu evidence for the default (frictional) workloads: launch lists C3/C2, --set full of the streamed k_pcg
# (C3) and the resident k_pcg_r (C2), raw csv + source pages
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/p_build.log 2>&1
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/p_smi.txt 2>&1
L="--no-e2e --no-schedule --no-cpu-baseline --no-alongside"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_c3.csv python bench.py --config C3 --steps 2 --warmup 3 $L > gpurun_out/p_launches_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_c2.csv python bench.py --config C2 --steps 2 --warmup 3 $L > gpurun_out/p_launches_c2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pcg\(" --launch-skip 0 --launch-count 1 -o /tmp/p_pcg_c3 -f python bench.py --config C3 --steps 1 --warmup 3 $L > gpurun_out/p_ncu_pcg_c3.log 2>&1
ncu -i /tmp/p_pcg_c3.ncu-rep --page raw --csv > gpurun_out/p_pcg_c3_raw.csv 2>/dev/null
ncu -i /tmp/p_pcg_c3.ncu-rep --page source --csv > gpurun_out/p_pcg_c3_source.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pcg_r\(" --launch-skip 0 --launch-count 1 -o /tmp/p_pcg_c2 -f python bench.py --config C2 --steps 1 --warmup 3 $L > gpurun_out/p_ncu_pcg_c2.log 2>&1
ncu -i /tmp/p_pcg_c2.ncu-rep --page raw --csv > gpurun_out/p_pcg_c2_raw.csv 2>/dev/null
