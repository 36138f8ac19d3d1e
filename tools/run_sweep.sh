for c in 3 4 6 8 12 16 24; do timeout 120 python tools/decode_probe.py perf 16 8 32 8192 $c; done
