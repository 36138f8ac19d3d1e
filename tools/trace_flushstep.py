"""Phases of one decode-time ring flush in flush_tc_kernel (CTA (0, 0, h), clock64 cycles):
setup (W tiles, TMEM, first images), the chunk, the S / P drain.  Tracing build:
    tools/trace_build.sh && KVLC_LIB=tools/_trace/libkvlinc.so python tools/trace_flushstep.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05373_b200 import _lib  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402

B, H, D = 16, 8, 128
bank = AdapterBank.initialize(H)
lib = _lib.load()
fn = lib["_ZN4kvlc16kvlc_ftrace_copyEPvm"]
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
for rep in range(2):
    c = BatchedKVCache(B, H, 32, 8192 + 512)
    k = torch.randn(B, H, 8064 + 255, D, device="cuda").bfloat16()
    c.prefill(k, k, adapters=bank)
    kt = torch.randn(B, H, D, device="cuda").bfloat16()
    torch.cuda.synchronize()
    c.append(kt, kt, adapters=bank)   # every sequence flushes one chunk (ring, tensor-core path)
    torch.cuda.synchronize()
buf = np.zeros((2, 40, 10), np.int64)
assert fn(buf.ctypes.data, buf.nbytes) == 0
for h in range(2):
    r = buf[h, 39]
    print(f"half {h}: setup {r[1] - r[0]} cyc, chunk {r[2] - r[1]} cyc, drain {r[3] - r[2]} cyc "
          f"(total {(r[3] - r[0]) / 1965:.1f} us at 1965 MHz)")
for h in range(2):
    st = buf[h, :2]  # per-chunk stamps of the first chunk: 0 start, 1 phi issued, 2 phi done, 3 softmax done, 4 S issued
    d = buf[h, 38]
    print(f"half {h}: chunk phases (cyc from chunk start) phi {st[0][1] - st[0][0]}, phi done {st[0][2] - st[0][0]}, "
          f"softmax done {st[0][3] - st[0][0]}, S issued {st[0][4] - st[0][0]}; drain: P {d[1] - d[0]}, "
          f"tile {d[2] - d[1]}, rows {d[3] - d[2]} cyc")
for h in range(2):
    st = buf[h, 0]
    print(f"half {h} softmax steps (cyc from chunk start): tmem ld {st[5] - st[0]}, max+sync {st[6] - st[0]}, "
          f"exp+sum+syncs {st[7] - st[0]}, hi/lo stores {st[8] - st[0]}, reduce-scatter {st[9] - st[0]}, done {st[3] - st[0]}")
