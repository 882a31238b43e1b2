# phase breakdown + launch list of one scheduled bench run + full ncu capture of k_pairs (bulk launch)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --phases --no-cpu-baseline --no-e2e > gpurun_out/bench_phases.log 2>&1; echo bench rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_s2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu-launch rc $?
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_pairs -c 1 -f -o gpurun_out/pairs_full python tools/pcg_traffic.py 1024 12 > gpurun_out/ncu_pairs.log 2>&1; echo ncu rc $?
tail -1 gpurun_out/bench_phases.log
