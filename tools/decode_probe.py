"""Quick GPU probe: decode precision vs the oracle and decode timing per shape.

    python tools/decode_probe.py prec          # max rel error vs oracle (fp16-meta cache)
    python tools/decode_probe.py perf B Hkv Hq N [cpw]
KVLC_EXTRA=0..3 selects the >4-head precision passes (see kvlc_decode.cu).
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402


def algo_bytes(B, Hkv, Hq, nq, nr, D=128, G=128, RANK=256):
    g = Hq // Hkv
    per_unit = 2 * nq * D // 4 + (nq // G) * D * 4 + nq * 4 + nr * D * 4 + D * RANK * 4 + RANK * 4 + g * D * 4
    return B * Hkv * per_unit + Hkv * 2 * D * (RANK // 2) * 4


def prec():
    from kvlc_testutil import bf16_round
    from oracle import kvlinc_oracle as orc
    for Hq, n in ((7, 640), (7, 4096), (8, 2000), (4, 4096)):
        g = orc.rng(n + Hq)
        k = bf16_round(g.standard_normal((1, 1, n, 128)).astype(np.float32))
        v = bf16_round(g.standard_normal((1, 1, n, 128)).astype(np.float32))
        q = bf16_round(g.standard_normal((1, Hq, 128)).astype(np.float32))
        td = lambda x: torch.from_numpy(x.astype(np.float32)).cuda().bfloat16()
        bank = AdapterBank.initialize(1)
        cache = BatchedKVCache(1, 1, Hq, n + 256)
        cache.prefill(td(k), td(v), adapters=bank)
        out = cache.decode(td(q), adapters=bank, out_dtype=torch.float32).cpu().numpy()
        oad = orc.init_adapter(128, 256, seed=0)
        oc = orc.fp16_meta_copy(orc.build_cache(k[0, 0], v[0, 0], oad))
        ref = np.stack([orc.decode_blocked(q[0, h], oc, oad) for h in range(Hq)])
        err = np.abs(out[0] - ref).max() / np.abs(ref).max()
        print(f"prec Hq={Hq} n={n} extra={os.environ.get('KVLC_EXTRA', 'default')} rel_err={err:.3e}")


def perf(B, Hkv, Hq, N, cpw=0):
    torch.manual_seed(0)
    reps = 4  # rotate caches so every step reads from HBM (4 x bytes > L2)
    caches = []
    bank = AdapterBank.initialize(Hkv)
    for r in range(reps):
        k = torch.randn(B, Hkv, N, 128, device="cuda").bfloat16()
        v = torch.randn(B, Hkv, N, 128, device="cuda").bfloat16()
        c = BatchedKVCache(B, Hkv, Hq, N + 256)
        c.prefill(k, v, adapters=bank)
        caches.append(c)
        del k, v
    q = torch.randn(B, Hq, 128, device="cuda").bfloat16()
    out = torch.empty_like(q)
    for c in caches:
        c.decode(q, adapters=bank, out=out, chunks_per_split=cpw)
    torch.cuda.synchronize()
    iters = 40
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        caches[i % reps].decode(q, adapters=bank, out=out, chunks_per_split=cpw)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    c = caches[0]
    nb = algo_bytes(B, Hkv, Hq, int(c.n_chunks[0]) * 128, int(c.res_len[0]))
    print(f"perf B={B} Hkv={Hkv} Hq={Hq} N={N} cpw={cpw} extra={os.environ.get('KVLC_EXTRA', 'default')}: "
          f"{us:.2f} us/step  {nb / 1e6:.2f} MB  {nb / us / 1e3:.0f} GB/s  ({nb / us / 1e3 / 6547.2 * 100:.1f}% of 6547)")


if __name__ == "__main__":
    if sys.argv[1] == "prec":
        prec()
    else:
        args = [int(x) for x in sys.argv[2:]]
        perf(*args)
