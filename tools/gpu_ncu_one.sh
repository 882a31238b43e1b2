# usage: bash tools/gpu_ncu_one.sh <kernel> [launch-skip]
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"^$1\$" --launch-skip ${2:-2} -c 1 -f -o gpurun_out/$1_full python tools/pcg_traffic.py 1024 12 > gpurun_out/ncu_$1.log 2>&1; echo $1 rc $?
