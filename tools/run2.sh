timeout 300 python tools/diag_probe.py 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:split_kernel -s 4 -c 1 -o gpurun_out/split_r1 python tools/decode_probe.py perf 16 8 32 8192 0 > gpurun_out/ncu_split_log.txt 2>&1
tail -3 gpurun_out/ncu_split_log.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 30 --csv --log-file gpurun_out/launches_r1.csv python tools/decode_probe.py perf 16 8 32 8192 0 > /dev/null 2>&1
tail -12 gpurun_out/launches_r1.csv
