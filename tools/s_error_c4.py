"""S / P error of one config-4 unit (131k tokens) vs the fp64 oracle."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
D, n = 128, 131072
g = orc.rng(2026)
k = torch.from_numpy(g.standard_normal((1, 8, n, D)).astype(np.float32)).bfloat16()
v = torch.from_numpy(g.standard_normal((1, 8, n, D)).astype(np.float32)).bfloat16()
c = BatchedKVCache(1, 8, 32, n + 256)
c.prefill(k.cuda(), v.cuda(), adapters=AdapterBank.initialize(8))
ad = orc.init_adapter(D, 256, seed=3)
oc = orc.build_cache(k[0, 3].float().numpy().astype(np.float64), v[0, 3].float().numpy().astype(np.float64), ad)
S = c.S[3].double().cpu().numpy()
print("S rel", np.linalg.norm(S - oc.s_state) / np.linalg.norm(oc.s_state))
