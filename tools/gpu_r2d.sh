#!/bin/bash
# state dumps for the preconditioner study (C2, C3), C5 AL diagnostic
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/d_build.log 2>&1
timeout 600 python tools/dump_states.py C3 8 40 5 > gpurun_out/d_dump_c3.log 2>&1
timeout 600 python tools/dump_states.py C2 8 60 5 > gpurun_out/d_dump_c2.log 2>&1
timeout 600 python tools/diag_c5.py 128 80 > gpurun_out/d_c5.log 2>&1
timeout 600 python tools/diag_c5.py 128 80 40 > gpurun_out/d_c5_al40.log 2>&1
