#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/d_build.log 2>&1
timeout 600 python tools/diag_c5.py 128 80 > gpurun_out/d_c5.log 2>&1
bash tools/gpu_prof_c3.sh
