timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in base qk3 qk4; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  echo "$v: $(KVLC_LIB=$L timeout 300 python tools/bench_prefill.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1), 'us')")"
done
