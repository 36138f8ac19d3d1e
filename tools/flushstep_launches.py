"""Kernels of one eager flushing step (config-2 shapes, all 128 units flush one chunk), for an
ncu launch list:  ncu --metrics gpu__time_duration.sum --csv python tools/flushstep_launches.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402

B, H, D = 16, 8, 128
bank = AdapterBank.initialize(H)
c = BatchedKVCache(B, H, 32, 8192 + 512)
k = torch.randn(B, H, 8064 + 255, D, device="cuda").bfloat16()
c.prefill(k, k, adapters=bank)
q = torch.randn(B, 32, D, device="cuda").bfloat16()
out = torch.empty_like(q)
c.decode(q, adapters=bank, out=out)
kt = torch.randn(B, H, D, device="cuda").bfloat16()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("flushstep")
c.append(kt, kt, adapters=bank)
c.decode(q, adapters=bank, out=out)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done")
