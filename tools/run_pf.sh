# prefill parity + config-5 timing (+ phase trace of the state kernel)
timeout 600 python -m pytest tests -m gpu -q -x -k "prefill or flush or batched or kvlc_io" 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/bench_prefill.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1), 'us')"; done
KVLC_LIB=tools/_trace/libkvlinc.so timeout 120 python tools/trace_prefill.py | head -8
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quant_kernel|flush_tc|reduce_state|prep_w" -c 8 --csv --log-file gpurun_out/launches_pf.csv python tools/bench_prefill.py --steps 1 --warmup 0 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launches_pf.csv
