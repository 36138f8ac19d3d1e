# interleaved same-box A/B of the default build against prebuilt variants in tools/_var/<name>, 3 rounds
for r in 1 2 3; do
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  KVLC_LIB=$L timeout 300 python bench.py --no-cpu --no-fa --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); o=d.get('other_configs',{})
print('$v', 'c2 step', round(d['us_per_step'],2), 'kernel', round(d['roofline']['split_us'],2),
      ' '.join(k.split('_')[0]+' '+str(round(x['us_per_step'],2)) for k,x in o.items() if isinstance(x, dict) and 'us_per_step' in x))"
done; done
