python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --profile-from-start off -k regex:k_pcg_r --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --print-units base --log-file gpurun_out/pcg_traffic.csv python tools/pcg_traffic.py 1024 12 > gpurun_out/pcg_traffic.log 2>&1; echo rc $?
python tools/pcg_traffic_summary.py gpurun_out/pcg_traffic.csv gpurun_out/pcg_traffic.log gpurun_out/pcg_traffic.json
