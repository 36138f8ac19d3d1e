tag=${1:-tc5}
bash tools/run_tc.sh $tag
KVLC_LIB=tools/_trace/libkvlinc.so timeout 120 python tools/trace_probe.py 2>&1 | head -22
