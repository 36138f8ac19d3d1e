"""Structure of the serving S-state error at config 4 (one 131k-token unit) vs the fp64 oracle:
relative Frobenius error, its rank-1 (channel-constant) part, its correlation with S, and P."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
D = 128
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
g = orc.rng(2026)
k = torch.from_numpy(g.standard_normal((1, 8, n, D)).astype(np.float32)).bfloat16()
v = torch.from_numpy(g.standard_normal((1, 8, n, D)).astype(np.float32)).bfloat16()
c = BatchedKVCache(1, 8, 32, n + 256)
c.prefill(k.cuda(), v.cuda(), adapters=AdapterBank.initialize(8))
ad = orc.init_adapter(D, 256, seed=3)
oc = orc.build_cache(k[0, 3].float().numpy().astype(np.float64), v[0, 3].float().numpy().astype(np.float64), ad)
S = c.S[3].double().cpu().numpy()
P = c.P[3].double().cpu().numpy()
R, RP = oc.s_state, oc.p_state
E = S - R
print(f"n={n} S rel {np.linalg.norm(E) / np.linalg.norm(R):.3e}  P rel {np.linalg.norm(P - RP) / np.linalg.norm(RP):.3e}")
col = E.mean(axis=0, keepdims=True)  # channel-constant (z^T Phi-like) part
print(f"rank-1 channel-constant part of E: {np.linalg.norm(np.broadcast_to(col, E.shape)) / np.linalg.norm(E):.3f} of ||E||")
print(f"corr(E, S_ref) = {(E * R).sum() / np.linalg.norm(E) / np.linalg.norm(R):+.3f}")
for h in range(2):
    Eh, Rh = E[:, 128 * h:128 * h + 128], R[:, 128 * h:128 * h + 128]
    print(f"half {h}: rel {np.linalg.norm(Eh) / np.linalg.norm(Rh):.3e}")
u, s_, vt = np.linalg.svd(E)
print("top singular values of E / ||E||:", np.round(s_[:5] / np.linalg.norm(E), 3))
