tag=${1:-tc6}
timeout 300 python -m pytest tests/test_gpu_batched.py -q -x -k split_partials 2>&1 | grep -E "AssertionError|rel diff|passed|failed" | head -5
bash tools/run_tc.sh $tag
KVLC_LIB=tools/_trace/libkvlinc.so timeout 120 python tools/trace_probe.py 2>&1 | head -18
