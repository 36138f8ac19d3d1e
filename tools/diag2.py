"""Per-chunk-range record check: decode_partial over [lo, hi) vs an exact oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from kvlc_testutil import bf16_round  # noqa: E402
from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200.batched import BatchedKVCache  # noqa: E402

LOG2E = 1.4426950408889634


def td(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().bfloat16()


Hq, n = (4, int(sys.argv[1])) if len(sys.argv) > 1 else (4, 128 * 9 + 128)
g = orc.rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
k = bf16_round(g.standard_normal((1, 1, n, 128)).astype(np.float32))
v = bf16_round(g.standard_normal((1, 1, n, 128)).astype(np.float32))
q = bf16_round(g.standard_normal((1, Hq, 128)).astype(np.float32))
cache = BatchedKVCache(1, 1, Hq, n + 256)
cache.prefill(td(k), td(v))
oc = orc.fp16_meta_copy(orc.build_cache(k[0, 0], v[0, 0], None))
print("chunks", cache.n_chunks)
nch = int(cache.n_chunks[0])
ranges = [(c, c + 1, 1) for c in range(nch)] + [(0, nch, 1), (0, nch, 8)]
for lo, hi, cpw in ranges:
    rec, _ = cache.decode_partial(td(q), lo, hi, False, chunks_per_split=cpw)
    rec = rec.cpu().numpy()[0]
    kh = oc.keys_dequant(lo * 128, hi * 128)
    vh = oc.values_dequant(lo * 128, hi * 128)
    errs = []
    for h in range(Hq):
        s = kh @ q[0, h] / np.sqrt(128)
        M = s.max()
        e = np.exp(s - M)
        y = e @ vh
        sc = np.exp(rec[h, 0] / LOG2E - M)
        errs.append(np.abs(rec[h, 4:132] * sc - y).max() / np.abs(y).max())
    print(f"[{lo},{hi}) cpw={cpw}: y rel err per head", " ".join(f"{x:.1e}" for x in errs))
