"""Phase timeline of the quantized-split CTAs (tracing build, tools/trace_build.sh).

    KVLC_LIB=tools/_trace/libkvlinc.so python tools/trace_probe.py [B Hkv Hq N]
Prints, for the first traced CTAs, the per-iteration cycle deltas between the
KVLC_STAMP points of kvlc_quant.cuh (token warp 0 / channel warp 4).
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05373_b200 import _lib  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402

B, Hkv, Hq, N = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (16, 8, 32, 8192)
torch.manual_seed(0)
bank = AdapterBank.initialize(Hkv)
k = torch.randn(B, Hkv, N, 128, device="cuda").bfloat16()
v = torch.randn(B, Hkv, N, 128, device="cuda").bfloat16()
cache = BatchedKVCache(B, Hkv, Hq, N + 256)
cache.prefill(k, v, adapters=bank)
q = torch.randn(B, Hq, 128, device="cuda").bfloat16()
for _ in range(3):
    cache.decode(q, adapters=bank)
torch.cuda.synchronize()
CT, K, P = 4, 32, 28
buf = np.zeros((CT, K + 1, P), dtype=np.int64)
lib = _lib.load()
lib.kvlc_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
rc = lib.kvlc_debug_trace(buf.ctypes.data, buf.nbytes)
assert rc == 0, rc
names_t = ["start", "kexp", "qk_wait", "frame", "softmax", "barrier", "issue"]
names_c = ["start", "pv_wait", "drain", "vexp", "bqk", "barrier", "issue"]
for cta in range(2):
    g = buf[cta, K]
    base = g[0]
    print(f"CTA {cta}: T setup {g[1]-base} | full0 wait {g[2]-g[1]} | prologue {g[3]-g[2]} | loop {g[4]-g[3]} | "
          f"teardown {g[5]-g[4]} ;  C setup {g[9]-g[8]} full0 {g[10]-g[9]} prologue {g[11]-g[10]} loop {g[12]-g[11]}")
    print("   k  T: " + " ".join(f"{n:>8s}" for n in names_t[1:]) + "  | C: " + " ".join(f"{n:>8s}" for n in names_c[1:]) + "   iter")
    for kk in range(K):
        r = buf[cta, kk]
        if r[0] == 0:
            break
        t = [r[i] - r[i - 1] if r[i] and r[i - 1] else -1 for i in range(1, 7)]
        cc = [r[i] - r[i - 1] if r[i] and r[i - 1] else -1 for i in range(9, 15)]
        it = buf[cta, kk + 1, 0] - r[0] if kk + 1 < K and buf[cta, kk + 1, 0] else -1
        arr = r[16:24]
        a0 = arr.min() if arr.min() > 0 else 0
        print(f"  {kk:2d}     " + " ".join(f"{x:8d}" for x in t) + "  |    " + " ".join(f"{x:8d}" for x in cc) + f"  {it:6d}"
              + "  arrive(w0..7 - first): " + " ".join(f"{x - a0:5d}" for x in arr)
              + f"  | C bar->fence {r[15]-r[13]} mma {r[25]-r[15]}")

# CTA timeline (globaltimer ns): per task type, start/end percentiles relative to the first CTA start
cta = np.zeros((4096, 4), dtype=np.uint64)
lib.kvlc_debug_cta.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.kvlc_debug_cta(cta.ctypes.data, cta.nbytes) == 0
used = cta[:, 0] > 0
c = cta[used].astype(np.int64)
t0 = c[:, 0].min()
print(f"CTAs {used.sum()}  kernel span {(c[:, 1].max() - t0) / 1e3:.1f} us")
for typ, name in ((0, "quant"), (1, "resid"), (2, "corr"), (3, "comb")):
    m = c[:, 3] == typ
    if not m.any():
        continue
    st, en = (c[m, 0] - t0) / 1e3, (c[m, 1] - t0) / 1e3
    du = en - st
    print(f"  {name:5s} n={m.sum():4d} start p0/50/100 {st.min():6.1f} {np.median(st):6.1f} {st.max():6.1f} us | "
          f"end p50/100 {np.median(en):6.1f} {en.max():6.1f} | dur p50/max {np.median(du):6.1f} {du.max():6.1f} us")
