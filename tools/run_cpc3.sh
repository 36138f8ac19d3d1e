for c in 0 6 7 8 9 10 11 12 14 16 20; do
  KVLC_CPC=$c timeout 300 python bench.py --no-cpu --no-fa --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('cpc $c', 'c2', round(d['us_per_step'],2), 'c3', round(d['other_configs']['config3_qwen2.5-7b_b16_ctx8k']['us_per_step'],2), 'c4', round(d['other_configs']['config4_llama3-8b_b1_ctx128k']['us_per_step'],2))"
done
