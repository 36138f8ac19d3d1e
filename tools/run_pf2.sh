tag=${1:-pf}
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python tools/bench_prefill.py
timeout 300 python tools/bench_prefill.py --batch 16 --tokens 8192
