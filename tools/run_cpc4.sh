for c in 16 20 22 24 28 32 40 48 64; do echo "cpc $c: $(timeout 120 python tools/decode_probe.py perf 1 8 32 131072 $c 2>&1 | tail -1 | cut -c1-90)"; done
