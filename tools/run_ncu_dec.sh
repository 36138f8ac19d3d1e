tag=${1:-dec}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:split_kernel -s 6 -c 1 -o gpurun_out/split_$tag python bench.py --steps 3 --warmup 3 --no-fa --no-cpu --no-extra > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log
python tools/ncu_summary.py gpurun_out/split_$tag.ncu-rep > gpurun_out/ncu_split_${tag}_summary.txt 2>&1
head -12 gpurun_out/ncu_split_${tag}_summary.txt
