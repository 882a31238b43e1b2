#!/bin/bash
# ncu --set full of the PCG kernels on the C2 bench (compaction on): the first launches of the timed
# steps include full-grid (iteration-0) launches; raw metrics exported to csv on the box
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/q_build.log 2>&1
B="python bench.py --config C2 --steps 2 --warmup 3 --no-e2e --no-schedule --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_cl --launch-skip 0 --launch-count 6 -o /tmp/q_pcgcl -f $B > gpurun_out/q_ncu1.log 2>&1
TAC_PCG_CLUSTER=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_r --launch-skip 0 --launch-count 6 -o /tmp/q_pcgr -f $B > gpurun_out/q_ncu2.log 2>&1
for r in q_pcgcl q_pcgr; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass > /dev/null 2>&1
done
cp /tmp/q_pcgcl.ncu-rep gpurun_out/ 2>/dev/null
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_contact.py -m gpu -q -rA > gpurun_out/q_tests.log 2>&1
