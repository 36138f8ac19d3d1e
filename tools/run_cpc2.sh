timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do
for c in 0 6 7 8 9 11; do
  KVLC_CPC=$c timeout 300 python bench.py --no-cpu --no-fa --no-extra --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('cpc $c', 'step', round(d['us_per_step'],2), 'kernel', round(d['roofline']['split_us'],2))"
done; done
