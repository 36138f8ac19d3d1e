# interleaved same-box A/B of environment settings on the default build, 3 rounds:
#   tools/run_abenv.sh "KVLC_X=0" "KVLC_X=1" ...   (each arg: space-separated VAR=value list)
for r in 1 2 3; do
for v in "$@"; do
  env $v timeout 300 python bench.py --no-cpu --no-fa --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); o=d.get('other_configs',{})
print('$v', 'c2 step', round(d['us_per_step'],2), 'kernel', round(d['roofline']['split_us'],2),
      ' '.join(k.split('_')[0]+' '+str(round(x['us_per_step'],2)) for k,x in o.items() if 'us_per_step' in x))"
done; done
