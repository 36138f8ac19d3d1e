# interleaved A/B of the default build against variants, 3 rounds (same box)
for r in 1 2 3; do
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  KVLC_LIB=$L timeout 300 python bench.py --no-cpu --no-fa --no-extra --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'step', round(d['us_per_step'],2), 'kernel', round(d['roofline']['split_us'],2))"
done; done
