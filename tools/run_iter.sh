# one iteration: gpu tests, bench line, qwen/128k probes, ncu capture of the split kernel
tag=${1:-it}
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','us_per_step')}, 'split_us', d['roofline']['split_us'], 'frac', d['roofline']['frac'], 'FA x', d['bf16_flash_attn']['speedup_ours_vs_fa'], d['clocks'])"
timeout 120 python tools/decode_probe.py perf 16 4 28 8192 0
timeout 120 python tools/decode_probe.py perf 1 8 32 131072 0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:split_kernel -s 6 -c 1 -o gpurun_out/split_$tag python bench.py --steps 3 --warmup 3 --no-fa --no-cpu > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log
