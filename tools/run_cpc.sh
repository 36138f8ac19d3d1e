bash tools/run_dec.sh "$@"
for c in 4 5 6 7 8 10 12 16; do echo "cpc $c: $(timeout 120 python tools/decode_probe.py perf 16 8 32 8192 $c 2>&1 | tail -1)"; done
