"""Relative Frobenius error of the prefill S / P states vs the fp64 oracle, by sequence length."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
D = 128
for n in (1024, 2048, 4096, 8192):
    g = orc.rng(77)
    k = torch.from_numpy(g.standard_normal((1, 1, n, D)).astype(np.float32)).bfloat16()
    v = torch.from_numpy(g.standard_normal((1, 1, n, D)).astype(np.float32)).bfloat16()
    c = BatchedKVCache(1, 1, 4, n + 256)
    c.prefill(k.cuda(), v.cuda(), adapters=AdapterBank.initialize(1, seeds=[0]))
    ad = orc.init_adapter(D, 256, seed=0)
    oc = orc.build_cache(k[0, 0].float().numpy().astype(np.float64), v[0, 0].float().numpy().astype(np.float64), ad)
    S, P = c.S[0].double().cpu().numpy(), c.P[0].double().cpu().numpy()
    rs = np.linalg.norm(S - oc.s_state) / np.linalg.norm(oc.s_state)
    rp = np.linalg.norm(P - oc.p_state) / np.linalg.norm(oc.p_state)
    print(f"n={n} chunks={len(oc.key_chunks)} S rel {rs:.2e} P rel {rp:.2e}")
