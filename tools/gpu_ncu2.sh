python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in k_broad k_pcg_r; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"^${k}\$" --launch-skip 2 -c 1 -f -o gpurun_out/${k}_full python tools/pcg_traffic.py 1024 12 > gpurun_out/ncu_${k}.log 2>&1; echo $k rc $?
done
bash tools/build_clocks.sh 2>/dev/null; cp paper_2504_12908_b200/libtaccel_cuda_clk.so paper_2504_12908_b200/libtaccel_cuda.so && touch paper_2504_12908_b200/libtaccel_cuda.so && python tools/pcg_clocks.py 1024 12 2 | head -12
