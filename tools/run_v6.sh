tag=${1:-v6}
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python bench.py --no-cpu > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -2 gpurun_out/bench_$tag.err
python -c "import json; d=json.load(open('gpurun_out/bench_$tag.json')); print('us', d['us_per_step'], 'split_us', d['roofline']['split_us'], 'frac', d['roofline']['frac'], 'FA x', d.get('bf16_flash_attn',{}).get('speedup_ours_vs_fa'), 'e2e', d['e2e']['value'], d['clocks'])"
timeout 120 python tools/decode_probe.py perf 16 4 28 8192 0
timeout 120 python tools/decode_probe.py perf 1 8 32 131072 0
