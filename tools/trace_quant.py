"""Per-CTA timeline of the ring-flush quant_kernel (config-2 flushing step, all 128 units).
Tracing build:  tools/build_variant.sh trace -DKVLC_TRACE
                KVLC_LIB=tools/_var/trace/libkvlinc.so python tools/trace_quant.py"""
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
try:
    fn = lib["_ZN4kvlc16kvlc_qtrace_copyEPvm"]
except Exception:
    fn = lib["kvlc_qtrace_copy"]
fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
for rep in range(2):
    c = BatchedKVCache(B, H, 32, 8192 + 512)
    k = torch.randn(B, H, 8064 + 255, D, device="cuda").bfloat16()
    c.prefill(k, k, adapters=bank)
    kt = torch.randn(B, H, D, device="cuda").bfloat16()
    torch.cuda.synchronize()
    buf = np.zeros((16, 128, 4), np.int64)
    c.append(kt, kt, adapters=bank)
    torch.cuda.synchronize()
assert fn(buf.ctypes.data, buf.nbytes) == 0
nz = int(np.nonzero(buf[:, 0, 0])[0].max()) + 1
t = buf[:nz]
t0 = t[:, :, 0].min()
for z in range(nz):
    s, k1, e = (t[z, :, 0] - t0) / 1e3, (t[z, :, 1] - t0) / 1e3, (t[z, :, 2] - t0) / 1e3
    print(f"z={z}: start [{s.min():6.2f} .. {s.max():6.2f}]  K1 part mean {np.mean(k1 - s):6.2f} max {np.max(k1 - s):6.2f}"
          f"  dur mean {np.mean(e - s):6.2f} max {np.max(e - s):6.2f}  end max {e.max():6.2f}  SMs {len(set(t[z, :, 3]))}")
tok = lib["_ZN4kvlc14kvlc_qtok_copyEPvm"]
tok.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
tb = np.zeros((128, 24, 2), np.int64)
assert tok(tb.ctypes.data, tb.nbytes) == 0
n = int((tb[0, :9, 0] > 0).sum())
dt = np.diff(tb[:, :n, 0], axis=1) / 1e3
lv = tb[:, 1:n, 1]
for L in (0, 1, 2):
    m = lv == L
    if m.any():
        print(f"tokens at level {L}: {m.sum():5d}  us per token mean {dt[m].mean():6.3f} max {dt[m].max():6.3f}")
print("first-token wait (us, from loop start):", np.round(dt[:, 0].mean(), 3))
ends = (tb[:, 9:17, 0] - tb[:, :1, 0]) / 1e3
print("per-warp loop end (us after warp 0 loop start) mean per warp:", np.round(ends.mean(0), 2), "max", np.round(ends.max(0), 2))
print("sync done", np.round(((tb[:, 17, 0] - tb[:, 0, 0]) / 1e3).mean(), 2), "CTA end", np.round(((tb[:, 18, 0] - tb[:, 0, 0]) / 1e3).mean(), 2))
lv = tb[:, 9:17, 1]
n1, n2 = lv & 255, lv >> 8
e = (tb[:, 9:17, 0] - tb[:, :1, 0]) / 1e3
for k in range(3):
    m = (n2 > 0) if k == 2 else ((n2 == 0) & (n1 > 0)) if k == 1 else ((n1 == 0) & (n2 == 0))
    if m.any():
        print(f"warps with {'dense' if k == 2 else 'fp64-FWHT' if k == 1 else 'no'} fallback: {m.sum():4d}  loop end mean {e[m].mean():6.2f} max {e[m].max():6.2f}")
d = (t[1, :, 2] - t[1, :, 0]) / 1e3
print("z=1 CTA duration percentiles 50/90/99/max:", np.round(np.percentile(d, [50, 90, 99, 100]), 2))
