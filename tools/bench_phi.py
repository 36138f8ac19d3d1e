"""In-step cost of phi_kernel / correction CTAs: config-2 decode graph replays with
and without adapters (4 rotating replicas as in bench.py)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402

B, HKV, HQ, CTX, D = 16, 8, 32, 8192, 128
bank = AdapterBank.initialize(HKV)
caches = []
for _ in range(4):
    c = BatchedKVCache(B, HKV, HQ, CTX + 256)
    k = torch.randn(B, HKV, CTX, D, device="cuda").bfloat16()
    c.prefill(k, k, adapters=bank)
    caches.append(c)
del k
q = torch.randn(B, HQ, D, device="cuda").bfloat16()
out = torch.empty_like(q)
for ad in (bank, None):
    for c in caches:
        c.decode(q, adapters=ad, out=out)
    graphs = [c.capture_decode(q, adapters=ad, out=out)[0] for c in caches]
    res = []
    for rep in range(3):
        for g in graphs:
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(100):
            graphs[i % 4].replay()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 10)
    print("adapters" if ad else "no-adapter", "step us", [round(x, 2) for x in res])
