# ncu --set full of the main kernels of one C2 step (step 12, 1024 envs)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in k_broad k_pcg_r k_assemble k_linesearch k_pairs_x; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"^${k}\$" --launch-skip 1 -c 1 -f -o gpurun_out/${k}_full python tools/pcg_traffic.py 1024 12 > gpurun_out/ncu_${k}.log 2>&1; echo $k rc $?
done
