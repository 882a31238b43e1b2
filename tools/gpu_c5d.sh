#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/d_build.log 2>&1
timeout 600 python tools/diag_c5.py 128 80 > gpurun_out/d_c5.log 2>&1
timeout 600 python tools/diag_c5.py 128 80 40 > gpurun_out/d_c5_al40.log 2>&1
