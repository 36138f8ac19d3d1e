tag=${1:-pfn}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flush_tc -c 1 -o gpurun_out/flushtc_$tag python tools/bench_prefill.py --steps 1 --warmup 0 > gpurun_out/ncu_flushtc_$tag.log 2>&1
tail -1 gpurun_out/ncu_flushtc_$tag.log
