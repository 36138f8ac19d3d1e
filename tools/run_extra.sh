for x in 0 1 2 3; do
  KVLC_EXTRA=$x timeout 300 python tools/decode_probe.py prec 2>&1 | grep prec
  KVLC_EXTRA=$x timeout 120 python tools/decode_probe.py perf 16 4 28 8192 2>&1 | tail -1 | cut -c1-100
done
