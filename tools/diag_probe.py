"""Locate decode error sources: quantized-part records vs an exact fp64 oracle,
tail-only caches, adapter on/off."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from kvlc_testutil import bf16_round  # noqa: E402
from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402

LOG2E = 1.4426950408889634


def td(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().bfloat16()


def run(Hq, n, use_ad):
    g = orc.rng(n + Hq)
    k = bf16_round(g.standard_normal((1, 1, n, 128)).astype(np.float32))
    v = bf16_round(g.standard_normal((1, 1, n, 128)).astype(np.float32))
    q = bf16_round(g.standard_normal((1, Hq, 128)).astype(np.float32))
    bank = AdapterBank.initialize(1) if use_ad else None
    oad = orc.init_adapter(128, 256, seed=0) if use_ad else None
    cache = BatchedKVCache(1, 1, Hq, n + 256)
    cache.prefill(td(k), td(v), adapters=bank)
    out = cache.decode(td(q), adapters=bank, out_dtype=torch.float32).cpu().numpy()[0]
    oc = orc.fp16_meta_copy(orc.build_cache(k[0, 0], v[0, 0], oad))
    ref = np.stack([orc.decode_blocked(q[0, h], oc, oad) for h in range(Hq)])
    dense = np.stack([orc.decode_dense(q[0, h], oc, oad) for h in range(Hq)])
    err = np.abs(out - ref).max() / np.abs(ref).max()
    err_d = np.abs(out - dense).max() / np.abs(dense).max()
    err_rd = np.abs(ref - dense).max() / np.abs(dense).max()
    print(f"Hq={Hq} n={n} ad={use_ad}: vs blocked {err:.2e}  vs dense {err_d:.2e}  "
          f"(blocked vs dense {err_rd:.2e})")
    nq = oc.quantized_tokens
    if nq:
        rec, _ = cache.decode_partial(td(q), 0, int(cache.n_chunks[0]), False)
        rec = rec.cpu().numpy()[0]
        kh = oc.keys_dequant(0, nq)
        vh = oc.values_dequant(0, nq)
        for h in range(min(Hq, 2)):
            s = kh @ q[0, h] / np.sqrt(128)
            M = s.max()
            e = np.exp(s - M)
            l, y = e.sum(), e @ vh
            m_got, l_got, y_got = rec[h, 0] / LOG2E, rec[h, 1], rec[h, 4:132]
            # compare after normalising to a common max
            scale = np.exp(m_got - M)
            print(f"   head {h}: m {m_got:.6f} vs {M:.6f}  l rel {abs(l_got * scale - l) / l:.2e}  "
                  f"y rel {np.abs(y_got * scale - y).max() / np.abs(y).max():.2e}")


if __name__ == "__main__":
    for Hq, n, ad in ((4, 4096, True), (4, 4096, False), (4, 200, False), (7, 4096, False),
                      (4, 640, False), (1, 8192, False)):
        run(Hq, n, ad)
