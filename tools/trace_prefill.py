"""Phase cycles of the tensor-core prefill flush (CTA (0, 0, h)); tracing build:
    KVLC_LIB=tools/_trace/libkvlinc.so python tools/trace_prefill.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05373_b200 import _lib  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402

B, Hkv, N = 1, 8, 32768
k = torch.randn(B, Hkv, N, 128, device="cuda").bfloat16()
v = torch.randn(B, Hkv, N, 128, device="cuda").bfloat16()
bank = AdapterBank.initialize(Hkv)
for _ in range(2):
    c = BatchedKVCache(B, Hkv, 32, N + 256)
    c.prefill(k, v, adapters=bank)
torch.cuda.synchronize()
lib = _lib.load()
buf = np.zeros((2, 40, 10), np.int64)
fn = lib["_ZN4kvlc16kvlc_ftrace_copyEPvm"]
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert fn(buf.ctypes.data, buf.nbytes) == 0
names = ["waitA+phi", "waitPhi+C+S", "softmax", "S+loadC"]
print("  it  " + " ".join(f"{n:>9s}" for n in names) + "   iter")
for it in range(12):
    r = buf[0, it]
    if r[0] == 0:
        break
    d = [r[i + 1] - r[i] for i in range(4)]
    nxt = buf[0, it + 1, 0] - r[0] if buf[0, it + 1, 0] else -1
    print(f"  {it:2d}  " + " ".join(f"{x:9d}" for x in d) + f"  {nxt:6d}")
