timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -25
for e in 0 1 2 3; do KVLC_EXTRA=$e timeout 120 python tools/decode_probe.py prec; done
python -c "import __graft_entry__ as g; g.smoke()"
