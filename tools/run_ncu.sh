# ncu full capture of the split kernel + launch list (1 GPU)
tag=${1:-ncu}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:split_kernel -s 6 -c 1 -o gpurun_out/split_$tag python bench.py --steps 3 --warmup 3 --no-fa --no-cpu > gpurun_out/ncu_$tag.log 2>&1
tail -2 gpurun_out/ncu_$tag.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 --no-fa --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_$tag.csv | head -8
