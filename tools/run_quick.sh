timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','us_per_step','e2e')}, d['roofline']['split_us'], d['roofline']['frac'], d.get('bf16_flash_attn'), d['clocks'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 3 --warmup 3 --no-fa --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_q.csv | head -8
