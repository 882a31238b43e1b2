#!/bin/bash
# C2/C3 bench + C3 launch list (kernel shares after the assembly split)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2504_12908_b200.build import build; build(force=True)" > gpurun_out/a_build.log 2>&1
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "pcg_matches or streamed or trajectory or chunked or 512" tests/test_gpu_contact.py > gpurun_out/a_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/a_tests.log
B="python bench.py --warmup 3 --no-e2e --no-cpu-baseline --no-alongside --no-schedule --phases"
timeout 600 $B --config C2 --steps 20 > gpurun_out/a_c2.json 2> gpurun_out/a_c2.err
timeout 900 $B --steps 10 > gpurun_out/a_c3.json 2> gpurun_out/a_c3.err
L="--no-e2e --no-schedule --no-cpu-baseline --no-alongside"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_launches_c3.csv python bench.py --config C3 --steps 2 --warmup 3 $L > gpurun_out/p_launches_c3.log 2>&1
