"""Per-step append cost of the serving cache (config-2 shapes, lockstep batch): plain appends
and the append that flushes every sequence (one chunk per (b, kv-head), adapters on)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
B, H, D = 16, 8, 128
bank = AdapterBank.initialize(H)
c = BatchedKVCache(B, H, 32, 8192 + 256)
k = torch.randn(B, H, 8064 + 255, D, device="cuda").bfloat16()
c.prefill(k, k, adapters=bank)          # residual window at 255: the next append flushes
kt = torch.randn(B, H, D, device="cuda").bfloat16()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); c.append(kt, kt, adapters=bank); e1.record(); torch.cuda.synchronize()
flush_us = e0.elapsed_time(e1) * 1e3
times = []
for i in range(20):
    e0.record(); c.append(kt, kt, adapters=bank); e1.record(); torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) * 1e3)
print(f"append with flush of all {B*H} units: {flush_us:.1f} us; plain append median {np.median(times):.1f} us;"
      f" amortised over 128 steps: {(flush_us - np.median(times)) / 128:.2f} us/step")
# device time of a plain append: captured once (all sequences active, none flushing)
c2 = BatchedKVCache(B, H, 32, 8192 + 256)
c2.prefill(k[:, :, :8064 + 10], k[:, :, :8064 + 10], adapters=bank)
c2.append(kt, kt, adapters=bank)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
res_len0 = c2.res_len.copy()
with torch.cuda.graph(g):
    c2.append(kt, kt, adapters=bank)
c2.res_len = res_len0  # host mirror: the capture did not run
torch.cuda.synchronize()
e0.record()
for _ in range(50):
    g.replay()
e1.record(); torch.cuda.synchronize()
print(f"graph-captured plain append (device): {e0.elapsed_time(e1) * 1e3 / 50:.2f} us")
import time
t0 = time.perf_counter()
for _ in range(50):
    c2.append(kt, kt, adapters=bank, active=np.ones(B, bool))
torch.cuda.synchronize()
print(f"host-side append call: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us")
