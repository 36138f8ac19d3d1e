# decode kernel variants: split-kernel time for config 2, and config 3 / 4 probes
for v in base $@; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  r=$(KVLC_LIB=$L timeout 300 python bench.py --no-cpu --no-fa --steps 30 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('us', round(d['us_per_step'],2), 'split', round(d['roofline']['split_us'],2), 'frac', round(d['roofline']['frac'],3))")
  q=$(KVLC_LIB=$L timeout 120 python tools/decode_probe.py perf 16 4 28 8192 0 2>/dev/null | grep -oE "[0-9.]+ us/step")
  l=$(KVLC_LIB=$L timeout 120 python tools/decode_probe.py perf 1 8 32 131072 0 2>/dev/null | grep -oE "[0-9.]+ us/step")
  echo "$v: cfg2 $r | qwen $q | 128k $l"
done
