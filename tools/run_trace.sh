KVLC_LIB=tools/_trace/libkvlinc.so python tools/trace_prefill.py
