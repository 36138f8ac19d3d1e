"""Per-CTA timeline of one fused decode launch (config 2 by default); tracing build:
    tools/trace_build.sh && KVLC_LIB=tools/_trace/libkvlinc.so python tools/trace_decode.py [B Hkv Hq ctx]
Prints, per task kind, start / work-end / exit times relative to the first CTA start (us)."""
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
k = torch.randn(B, Hkv, N, 128, device="cuda").bfloat16()
v = torch.randn(B, Hkv, N, 128, device="cuda").bfloat16()
q = torch.randn(B, Hq, 128, device="cuda").bfloat16()
bank = AdapterBank.initialize(Hkv)
c = BatchedKVCache(B, Hkv, Hq, N + 256)
c.prefill(k, v, adapters=bank)
for _ in range(20):
    c.decode(q, adapters=bank)
torch.cuda.synchronize()
lib = _lib.load()
fn = lib["kvlc_dtrace_copy"]
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
buf = np.zeros((8192, 4), np.uint64)
assert fn(buf.ctypes.data, buf.nbytes) == 0
n = int(np.nonzero(buf[:, 0])[0].max()) + 1
t = buf[:n].astype(np.int64)
comb = (buf[:n, 2] >> np.uint64(63)).astype(bool)
t2 = (buf[:n, 2] & np.uint64((1 << 63) - 1)).astype(np.int64)
t0 = t[:, 0].min()
start, work, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t2 - t0) / 1e3
kind = ((buf[:n, 3] >> np.uint64(24)) & np.uint64(0xff)).astype(int)
sm = (buf[:n, 3] >> np.uint64(32)).astype(int)
print(f"CTAs {n}, span {end.max():.2f} us, SMs used {len(set(sm))}")
for kd, name in enumerate(["correction", "split", "residual"]):
    m = kind == kd
    if not m.any():
        continue
    d = work[m] - start[m]
    print(f"{name:10s} n={m.sum():5d} start [{start[m].min():6.2f} .. {start[m].max():6.2f}]"
          f" dur mean {d.mean():6.2f} min {d.min():6.2f} max {d.max():6.2f}"
          f"  work-end max {work[m].max():6.2f}  exit max {end[m].max():6.2f}")
if comb.any():
    cd = end[comb] - work[comb]
    print(f"combine CTAs {comb.sum()}: combine dur mean {cd.mean():.2f} max {cd.max():.2f}, "
          f"last combine ends {end[comb].max():.2f}")
# which kind finishes last per unit (the unit's critical task)
hist = np.histogram(end, bins=np.arange(0, end.max() + 2, 2.0))[0]
print("exits per 2 us:", " ".join(str(x) for x in hist))
act = [int(((start <= x) & (end > x)).sum()) for x in np.arange(0, end.max(), 2.0)]
print("resident CTAs per 2 us:", " ".join(str(x) for x in act))
np.save(os.path.join(ROOT, "gpurun_out", "dtrace.npy"), np.stack([start, work, end, kind, sm, comb], 1))
# phase stamps (PH_STAMP): correction 0 after griddepcontrol.wait, 1 q staged, 2 phi done;
# split 0 after the wait, 1 q staged, 2 chunks done; relative to the CTA start
try:
    fp = lib["kvlc_dphase_copy"]
    fp.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    ph = np.zeros((8192, 4), np.uint64)
    assert fp(ph.ctypes.data, ph.nbytes) == 0
    ph = ph[:n].astype(np.int64)
    for kd, name in enumerate(["correction", "split"]):
        m = kind == kd
        if not m.any():
            continue
        rel = (ph[m, :3] - t[m, 0:1]) / 1e3
        print(f"{name:10s} phases (us from CTA start, mean / max): " +
              "  ".join(f"p{k} {rel[:, k].mean():6.2f}/{rel[:, k].max():6.2f}" for k in range(3)))
except (KeyError, AttributeError):
    pass
