#!/bin/bash
# round-2 end evidence: GPU tests, default bench (C3 + C2 alongside, e2e, CPU baseline), C4/C5 lines, ncu launch
# lists, ncu --set full of the PCG kernels, PCG DRAM traffic per launch, compute-sanitizer on the sanity workload
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f_smi.txt 2>&1
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/f_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=30 > gpurun_out/f_gputest.log 2>&1
echo "pytest exit $?" >> gpurun_out/f_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/f_smoke.log
timeout 1500 python bench.py --phases > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 900 python bench.py --config C4 --phases --no-cpu-baseline > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
timeout 900 python bench.py --config C5 --phases --no-cpu-baseline > gpurun_out/f_bench_c5.json 2> gpurun_out/f_bench_c5.err
L="--no-e2e --no-schedule --no-cpu-baseline --no-alongside"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_c3.csv python bench.py --config C3 --steps 2 --warmup 3 $L > gpurun_out/f_launches_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_c2.csv python bench.py --config C2 --steps 2 --warmup 3 $L > gpurun_out/f_launches_c2.log 2>&1
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
timeout 900 ncu --profile-from-start off -k regex:"^k_pcg" $M --csv --log-file gpurun_out/f_traffic_c3.csv python tools/pcg_traffic.py C3 4096 5 > gpurun_out/f_traffic_c3.log 2>&1
timeout 600 ncu --profile-from-start off -k regex:"^k_pcg" $M --csv --log-file gpurun_out/f_traffic_c2.csv python tools/pcg_traffic.py C2 1024 12 > gpurun_out/f_traffic_c2.log 2>&1
# full-set captures at 1024 envs (C3 x 4096 makes ncu back the device memory up in host memory and fail)
for K in "^k_pcg:k_pcg:C3" "^k_pcg_r$:k_pcg_r:C2" "^k_assemble_soft$:k_assemble_soft:C3" "^k_asm_edges$:k_asm_edges:C3"; do
  RX=$(echo $K | cut -d: -f1); TAG=$(echo $K | cut -d: -f2); CF=$(echo $K | cut -d: -f3)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${RX}" --launch-skip 0 --launch-count 1 -o /tmp/f_${TAG}_${CF} -f python bench.py --config $CF --envs-total 1024 --steps 1 --warmup 3 $L > gpurun_out/f_ncu_${TAG}_${CF}.log 2>&1
  ncu -i /tmp/f_${TAG}_${CF}.ncu-rep --page raw --csv > gpurun_out/f_${TAG}_${CF}_raw.csv 2>/dev/null
done
# compute-sanitizer is closed on this GPU pool (its runs left GPUs needing a reset)
