# interleaved same-box A/B of environment settings over config 1 and the config-3 sweep, 2 rounds:
#   tools/run_absweep.sh "KVLC_X=0" "KVLC_X=1" ...
for r in 1 2; do
for v in "$@"; do
  env $v timeout 300 python bench.py --no-cpu --no-fa --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); o=d.get('other_configs',{})
sw=o.get('config3_sweep_qwen2.5-7b',{})
print('$v', 'c2', round(d['us_per_step'],2), 'c1', [round(x['us_per_step'],2) for k,x in o.items() if k.startswith('config1')],
      ' '.join(k+' '+str(round(x['us_per_step'],2)) for k,x in sw.items()))"
done; done
