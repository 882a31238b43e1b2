#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/d_build.log 2>&1
timeout 600 python tools/diag_c5.py 128 40 > gpurun_out/d_c5.log 2>&1
timeout 600 python tools/dbg_r2.py trace C3 38 8 > gpurun_out/d_trace_c3.log 2>&1
timeout 600 python tools/dbg_r2.py trace C2 40 1024 > gpurun_out/d_trace_c2.log 2>&1
