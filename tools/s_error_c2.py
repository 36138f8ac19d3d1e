"""S error of a sampled unit in a 128-unit 8k prefill (config-2 shapes) vs the fp64 oracle."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
D, n, B, H = 128, 8192, 16, 8
g = orc.rng(2024)
k = torch.from_numpy(g.standard_normal((B, H, n, D)).astype(np.float32)).bfloat16()
v = torch.from_numpy(g.standard_normal((B, H, n, D)).astype(np.float32)).bfloat16()
c = BatchedKVCache(B, H, 32, n + 256)
c.prefill(k.cuda(), v.cuda(), adapters=AdapterBank.initialize(H))
for (b, h) in ((0, 0), (7, 7)):
    ad = orc.init_adapter(D, 256, seed=h)
    oc = orc.build_cache(k[b, h].float().numpy().astype(np.float64), v[b, h].float().numpy().astype(np.float64), ad)
    S = c.S[b * H + h].double().cpu().numpy()
    print((b, h), "S rel", np.linalg.norm(S - oc.s_state) / np.linalg.norm(oc.s_state))
