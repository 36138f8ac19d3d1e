# decode parity + config-2 step / kernel / e2e for the default build and variants in tools/_var/
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  KVLC_LIB=$L timeout 300 python bench.py --no-cpu --no-fa --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'step', round(d['us_per_step'],2), 'kernel', round(d['roofline']['split_us'],2), 'e2e', round(d['e2e']['ms_per_step']*1e3,2), {k[:7]: round(v['us_per_step'],1) for k,v in d['other_configs'].items()})"
done
