# ncu full capture of the prefill kernels (quant_kernel, flush_tc_kernel) on config 5
tag=${1:-pf}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"quant_kernel|flush_tc_kernel" -s 2 -c 2 -o gpurun_out/prefill_$tag python tools/bench_prefill.py --steps 1 --warmup 1 > gpurun_out/ncu_$tag.log 2>&1
tail -2 gpurun_out/ncu_$tag.log
