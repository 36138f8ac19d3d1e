tag=${1:-pf}
timeout 300 python tools/bench_prefill.py
timeout 300 python tools/bench_prefill.py --no-adapter
timeout 600 ncu --set full --clock-control none --import-source on -k regex:flush_kernel -c 1 -o gpurun_out/flush_$tag python tools/bench_prefill.py --steps 1 --warmup 0 > gpurun_out/ncu_flush_$tag.log 2>&1
tail -1 gpurun_out/ncu_flush_$tag.log
