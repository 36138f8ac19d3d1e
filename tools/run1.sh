set -x
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -5
for e in 0 1 2 3; do KVLC_EXTRA=$e timeout 120 python tools/decode_probe.py prec; done
for c in 1 2 4; do timeout 120 python tools/decode_probe.py perf 16 8 32 8192 $c; done
timeout 120 python tools/decode_probe.py perf 16 8 32 8192 0
for e in 0 3; do KVLC_EXTRA=$e timeout 120 python tools/decode_probe.py perf 16 4 28 8192 0; done
timeout 120 python tools/decode_probe.py perf 1 8 32 131072 0
