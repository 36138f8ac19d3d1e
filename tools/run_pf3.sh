timeout 600 python -m pytest tests/test_gpu_batched.py -q -x -k "prefill_and_decode" 2>&1 | grep -E "^E|test_gpu_batched.py:[0-9]+|passed|failed" | head -20
