# Warp-per-chunk split sweeps: chunks per split x correction CTAs per unit (configs 2-4)
for cs in 0 1 2; do
for c in 0 8 12 16 20 24; do
  KVLC_CORRSPLIT=$cs KVLC_CPC=$c timeout 300 python bench.py --no-cpu --no-fa --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('corrsplit $cs cpc $c', 'c2', round(d['us_per_step'],2), round(d['roofline']['split_us'],2), 'c3', round(d['other_configs']['config3_qwen2.5-7b_b16_ctx8k']['us_per_step'],2), 'c4', round(d['other_configs']['config4_llama3-8b_b1_ctx128k']['us_per_step'],2))"
done
done
