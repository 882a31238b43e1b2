# round-end evidence: smoke, GPU tests, default bench line, launch list of the bench command, PCG traffic
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc $?
timeout 900 python bench.py --phases --no-cpu-baseline --no-e2e > gpurun_out/bench_phases.log 2>&1; echo bench-phases rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu-launch rc $?
timeout 900 ncu --profile-from-start off -k regex:k_pcg_r --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --print-units base --log-file gpurun_out/pcg_traffic.csv python tools/pcg_traffic.py 1024 12 > gpurun_out/pcg_traffic.log 2>&1; echo traffic rc $?
python tools/pcg_traffic_summary.py gpurun_out/pcg_traffic.csv gpurun_out/pcg_traffic.log gpurun_out/pcg_traffic.json > /dev/null
for k in k_pcg_r k_pairs_x k_broad; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"^${k}\$" --launch-skip 2 -c 1 -f -o gpurun_out/${k}_full python tools/pcg_traffic.py 1024 12 > gpurun_out/ncu_${k}.log 2>&1; echo $k rc $?
done
tail -1 gpurun_out/bench.log
