# A/B of the PCG register budgets: k_pcg_r at 384-thread bounds (default) vs 512
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.log 2>&1
for v in 0 1; do
  TAC_PCG_R_LB512=$v timeout 600 python bench.py --phases --no-cpu-baseline --no-e2e > gpurun_out/ab_c2_lb512_$v.log 2>&1; echo c2 lb512=$v rc $?
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest rc $?; tail -1 gpurun_out/ab_pytest.log
for f in gpurun_out/ab_c*.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v['ms'],1) for k,v in d['phases'].items() if k=='pcg'})"; done
