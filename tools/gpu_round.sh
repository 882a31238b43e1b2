set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc $?
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_pcg -c 1 -f -o gpurun_out/pcg_full python tools/pcg_traffic.py 1024 12 > gpurun_out/ncu_full.log 2>&1; echo ncu rc $?
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.log | tail -2
