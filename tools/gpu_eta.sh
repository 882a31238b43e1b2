#!/bin/bash
# PCG tolerance sweep (reading R15's eta): C3 and C2 throughput and Newton / PCG counts
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/a_build.log 2>&1
B="python bench.py --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --no-schedule"
for eta in 3e-4 1e-3; do
  timeout 900 $B --steps 10 --set pcg_eta=$eta > gpurun_out/eta_c3_$eta.json 2> gpurun_out/eta_c3_$eta.err
  timeout 600 $B --config C2 --steps 20 --set pcg_eta=$eta > gpurun_out/eta_c2_$eta.json 2> gpurun_out/eta_c2_$eta.err
done
