for r in 1 2; do for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  echo "$v $(KVLC_LIB=$L python tools/bench_prefill.py | grep -o 'us_per_step": [0-9.]*')"
done; done
