#!/bin/bash
# round-2 evidence: bench lines (C3 primary + C2, C4, C5, C2 with friction), ncu launch lists, ncu --set full
# of the PCG kernels (+ DRAM traffic), compute-sanitizer runs.  Outputs in gpurun_out/ev_*.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/ev_build.log 2>&1
timeout 1500 python bench.py --phases > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 900 python bench.py --config C4 --phases --no-cpu-baseline > gpurun_out/ev_bench_c4.json 2> gpurun_out/ev_bench_c4.err
timeout 900 python bench.py --config C5 --phases --no-cpu-baseline > gpurun_out/ev_bench_c5.json 2> gpurun_out/ev_bench_c5.err
timeout 600 python bench.py --config C2 --set mu_friction=0.5 --phases --no-cpu-baseline > gpurun_out/ev_bench_c2_friction.json 2> gpurun_out/ev_bench_c2_friction.err
L="--no-e2e --no-schedule --no-cpu-baseline --no-alongside"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c3.csv python bench.py --config C3 --steps 2 --warmup 3 $L > gpurun_out/ev_launches_c3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c2.csv python bench.py --config C2 --steps 2 --warmup 3 $L > gpurun_out/ev_launches_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pcg\(" --launch-skip 0 --launch-count 1 -o /tmp/ev_pcg_c3 -f python bench.py --config C3 --steps 1 --warmup 3 $L > gpurun_out/ev_ncu_pcg_c3.log 2>&1
ncu -i /tmp/ev_pcg_c3.ncu-rep --page raw --csv > gpurun_out/ev_pcg_c3_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pcg_r\(" --launch-skip 0 --launch-count 1 -o /tmp/ev_pcg_c2 -f python bench.py --config C2 --steps 1 --warmup 3 $L > gpurun_out/ev_ncu_pcg_c2.log 2>&1
ncu -i /tmp/ev_pcg_c2.ncu-rep --page raw --csv > gpurun_out/ev_pcg_c2_raw.csv 2>/dev/null
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/dbg_r2.py sanity > gpurun_out/ev_sanitizer_$tool.log 2>&1
done
