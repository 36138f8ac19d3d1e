"""Decode-output error decomposition on one unit vs the oracle (tools only):
adapter off / on, and on with the oracle's S, P replaced by the GPU's (isolates the state error)."""
import copy, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
D = 128
B, Hkv, Hq, n, seed = (int(x) for x in sys.argv[1:6]) if len(sys.argv) > 5 else (1, 4, 28, 32768, 2028)
g = orc.rng(seed)
bf = lambda s: torch.from_numpy(g.standard_normal(s).astype(np.float32)).bfloat16()
k, v, q = bf((B, Hkv, n, D)), bf((B, Hkv, n, D)), bf((B, Hq, D))
NG = Hq // Hkv
seeds = list(range(Hkv))
bank = AdapterBank.initialize(Hkv, seeds=seeds)
c = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
c.prefill(k.cuda(), v.cuda(), adapters=bank)
out_on = c.decode(q.cuda(), adapters=bank, out_dtype=torch.float32).cpu().numpy()
out_off = c.decode(q.cuda(), adapters=None, out_dtype=torch.float32).cpu().numpy()
b, h = 0, 0
ad = orc.init_adapter(D, 256, seed=seeds[h])
oc = orc.build_cache(k[b, h].float().numpy().astype(np.float64), v[b, h].float().numpy().astype(np.float64), ad)
ocm = orc.fp16_meta_copy(oc)
ocg = copy.deepcopy(ocm)
ocg.s_state = c.S[b * Hkv + h].double().cpu().numpy()
ocg.p_state = c.P[b * Hkv + h].double().cpu().numpy()
qn = q.float().numpy().astype(np.float64)
for i in range(NG):
    qq = qn[b, h * NG + i]
    r_off = orc.decode_blocked(qq, ocm, None)
    r_on = orc.decode_blocked(qq, ocm, ad)
    r_ong = orc.decode_blocked(qq, ocg, ad)
    e = lambda o, r: np.abs(o - r).max() / np.abs(r).max()
    print(f"head {i}: off {e(out_off[b, h * NG + i], r_off):.2e}  on {e(out_on[b, h * NG + i], r_on):.2e}  "
          f"on-vs-oracle-with-gpu-S {e(out_on[b, h * NG + i], r_ong):.2e}  max|ref| on {np.abs(r_on).max():.3e} off {np.abs(r_off).max():.3e}")
# structure of the error of head 0 (adapter off): raw channels and rotated basis (H e)
H = orc.hadamard(D) if hasattr(orc, "hadamard") else None
qq = qn[b, h * NG]
r_off = orc.decode_blocked(qq, ocm, None)
err = out_off[b, h * NG] - r_off
print("err raw: max", np.abs(err).max(), "mean", err.mean(), "top idx", np.argsort(-np.abs(err))[:6])
if H is not None:
    er = H @ err
    print("err rotated: top idx", np.argsort(-np.abs(er))[:6], "vals", np.round(er[np.argsort(-np.abs(er))[:6]], 7))
np.savez(os.path.join(ROOT, "gpurun_out", f"dec_diag_{n}.npz"), out_off=out_off[b, h * NG:(h + 1) * NG],
         ref_off=np.stack([orc.decode_blocked(qn[b, h * NG + i], ocm, None) for i in range(NG)]))
