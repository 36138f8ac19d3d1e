# interleaved A/B on configs 2-4 (bench other_configs), 2 rounds
for r in 1 2; do
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L="tools/_var/$v/libkvlinc.so"; fi
  KVLC_LIB=$L timeout 300 python bench.py --no-cpu --no-fa --steps 100 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'c2', round(d['us_per_step'],2), 'k', round(d['roofline']['split_us'],2), 'c3', round(d['other_configs']['config3_qwen2.5-7b_b16_ctx8k']['us_per_step'],2), 'c4', round(d['other_configs']['config4_llama3-8b_b1_ctx128k']['us_per_step'],2))"
done; done
