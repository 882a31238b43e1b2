# parity suite + phase-split bench (no e2e / cpu baseline)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --phases --no-cpu-baseline --no-e2e > gpurun_out/bench_phases.log 2>&1; echo bench rc $?
tail -1 gpurun_out/bench_phases.log
