# parity of the prefill paths + config-5 timing for the default build and variants in tools/_var/
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  echo "== $v: $(KVLC_LIB=$L timeout 600 python -m pytest tests -m gpu -q -x -k "prefill or flush or batched" 2>&1 | tail -1)"
  echo "   $(KVLC_LIB=$L timeout 300 python tools/bench_prefill.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],1), 'us')")"
done
