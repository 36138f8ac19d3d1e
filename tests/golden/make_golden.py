"""Generate the golden fixtures that pin the oracle (and through it the CUDA
path) to the REFERENCE implementation.

Runs the reference package itself (read-only tree at /root/reference, which
exists only in the build container, never on the GPU box) and stores its
outputs as compressed .npz files next to this script:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Inputs are regenerated from seeds with the reference's own PCG64 `rng`
(linalg.py:16-18), so every fixture is reproducible.  Shapes follow the
reference's unit / acceptance tests (test_quantize.py, test_cache.py,
test_attention.py, test_acceptance.py:115-137) plus the d=128 / G=128 /
R=128 / D=256 production shape the fast kernels specialise on.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

from quantkv.adapter import (CorrectionAdapter, TrainSettings, _batched_loss_and_grads,  # noqa: E402
                             corrected_weights, feature_map, loss_and_grads, phi_k, phi_q,
                             serialize_adapter, train_adapter)
from quantkv.attention import (OpCounter, attention_reference,  # noqa: E402
                               corrected_attention_quadratic, corrected_attention_recurrent,
                               decode_step_blocked)
from quantkv.cache import KVCacheState, memory_footprint, serialize_cache  # noqa: E402
from quantkv.hadamard import hadamard_matrix, rotate  # noqa: E402
from quantkv.linalg import rng  # noqa: E402
from quantkv.quantize import (QuantConfig, pack_codes, quantize_group,  # noqa: E402
                              quantize_tensor, unpack_codes)

HERE = os.path.dirname(os.path.abspath(__file__))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 -> fp64 (the serving path's inputs)."""
    f = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    rounded = ((f + 0x7FFF + ((f >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32).astype(np.float64)


def quantize_cases():
    out = {}
    cases = [  # (name, rows, cols, bits, group, axis, seed, kind)
        ("tok_2b_g32", 128, 64, 2, 32, "token", 3, "normal5"),
        ("chan_2b_g32", 128, 64, 2, 32, "channel", 3, "normal5"),
        ("chan_2b_g128", 256, 8, 2, 128, "channel", 2, "normal"),
        ("tok_short", 3, 10, 2, 4, "token", 4, "normal"),
        ("tok_3b", 17, 37, 3, 8, "token", 11, "normal"),
        ("tok_4b", 9, 50, 4, 16, "token", 12, "normal"),
        ("chan_8b", 40, 12, 8, 16, "channel", 13, "normal"),
        ("chan_prod", 128, 128, 2, 128, "channel", 14, "bf16"),
        ("tok_prod", 128, 128, 2, 128, "token", 15, "bf16"),
        ("tok_ties", 64, 16, 2, 16, "token", 16, "grid"),
        ("chan_const", 32, 8, 2, 32, "channel", 17, "const"),
    ]
    for name, r, c, bits, g, axis, seed, kind in cases:
        gen = rng(seed)
        if kind == "normal5":
            x = gen.standard_normal((r, c)) * 5
        elif kind == "bf16":
            x = bf16_round(gen.standard_normal((r, c)).astype(np.float32))
        elif kind == "grid":  # exact .5 ties after (x-min)/scale
            x = gen.integers(0, 7, size=(r, c)).astype(np.float64) * 0.5
            x[:, 0] = 0.0
            x[:, 1] = 3.0
        elif kind == "const":
            x = np.repeat(gen.standard_normal((1, c)), r, axis=0)
            x[:, :3] = gen.standard_normal((r, 3))
        else:
            x = gen.standard_normal((r, c))
        qt = quantize_tensor(x, QuantConfig(bits=bits, group_size=g, axis=axis))
        out[f"{name}/x"] = x
        out[f"{name}/codes"] = qt.codes.astype(np.uint32)
        out[f"{name}/scales"] = qt.scales
        out[f"{name}/zeros"] = qt.zeros
        out[f"{name}/deq"] = qt.dequantize()
        out[f"{name}/meta"] = np.array([r, c, bits, g, 0 if axis == "token" else 1])
    # known answers (test_quantize.py:24-28, 85-89)
    codes, scale, zero = quantize_group([0.0, 0.5, 1.5, 3.0], bits=2)
    out["ka/half_even_codes"] = codes
    out["ka/half_even_scale"] = np.array([scale, zero])
    out["ka/lane_word"] = pack_codes(np.array([3, 2, 1, 0] + [0] * 12), bits=2)
    gen = rng(1)
    codes = gen.integers(0, 4, size=(5, 37))
    out["ka/pack_rows_codes"] = codes.astype(np.uint8)
    out["ka/pack_rows_words"] = pack_codes(codes, bits=2)
    for bits in (2, 3, 4, 8):
        c = gen.integers(0, 1 << bits, size=(3, 41))
        out[f"ka/pack_{bits}b_codes"] = c.astype(np.uint8)
        out[f"ka/pack_{bits}b_words"] = pack_codes(c, bits)
        assert np.array_equal(unpack_codes(out[f"ka/pack_{bits}b_words"], 41, bits), c)
    return out


def hadamard_cases():
    out = {}
    for dim in (2, 4, 8, 16, 32, 64, 128, 256):
        out[f"H/{dim}"] = hadamard_matrix(dim).matrix
    gen = rng(7)
    for dim in (16, 64, 128):
        x = gen.standard_normal((24, dim)) * 3
        out[f"rot/post_{dim}/x"] = x
        out[f"rot/post_{dim}/y"] = rotate(x, hadamard_matrix(dim), "post")
    x = gen.standard_normal((32, 8))
    out["rot/pre_32/x"] = x
    out["rot/pre_32/y"] = rotate(x, hadamard_matrix(32), "pre")
    return out


def adapter_cases():
    out = {}
    for d, rank, seed in ((4, 8, 0), (16, 8, 3), (64, 32, 2), (128, 256, 0), (128, 256, 5)):
        ad = CorrectionAdapter.initialize(d, rank, seed=seed)
        key = f"ad/{d}_{rank}_{seed}"
        for n in ("w1_q", "w2_q", "w1_k", "w2_k"):
            out[f"{key}/{n}"] = getattr(ad, n)
        x = rng(seed + 100).standard_normal((6, d)) * 2
        out[f"{key}/x"] = x
        out[f"{key}/phi_q"] = phi_q(ad, x)
        out[f"{key}/phi_k"] = phi_k(ad, x)
        out[f"{key}/fm_vec"] = feature_map(x[0], ad.w1_q, ad.w2_q)
    return out


CACHE_CASES = [  # name, n, d, group, window, rotate, rank(0=none), adapter seed, data seed, bf16
    ("c_small", 80, 16, 32, 16, False, 8, 3, 4, False),
    ("c_rot", 256, 32, 64, 0, True, 16, 7, 8, False),
    ("c_lit", 64, 8, 32, 0, False, 8, 9, 13, False),
    ("c_acc129", 129, 64, 128, 0, False, 32, 2, 129, False),
    ("c_acc512", 512, 64, 128, 128, False, 32, 2, 512, False),
    ("c_rot_win", 200, 16, 32, 24, True, 8, 1, 21, False),
    ("c_noad", 300, 32, 64, 32, True, 0, 0, 22, False),
    ("c_prod", 640, 128, 128, 128, True, 256, 0, 23, True),
]


def cache_cases():
    out = {}
    for name, n, d, g, win, rot, rank, aseed, dseed, bf16 in CACHE_CASES:
        gen = rng(dseed)
        k = gen.standard_normal((n, d))
        v = gen.standard_normal((n, d))
        if bf16:
            k, v = bf16_round(k), bf16_round(v)
        ad = CorrectionAdapter.initialize(d, rank, seed=aseed) if rank else None
        cache = KVCacheState(d, group_size=g, residual_window=win, rotate_values=rot)
        for t in range(n):
            cache.append(k[t], v[t], ad)
        p = f"{name}/"
        out[p + "k"] = k
        out[p + "v"] = v
        out[p + "meta"] = np.array([n, d, g, win, int(rot), rank, aseed,
                                    cache.quantized_tokens, cache.residual_len,
                                    cache.tokens_total])
        if cache.key_chunks:
            out[p + "kcodes"] = np.stack([c.codes for c in cache.key_chunks])
            out[p + "kscales"] = np.stack([c.scales for c in cache.key_chunks])
            out[p + "kzeros"] = np.stack([c.zeros for c in cache.key_chunks])
            out[p + "vcodes"] = cache.value_rows.codes
            out[p + "vscales"] = cache.value_rows.scales
            out[p + "vzeros"] = cache.value_rows.zeros
        out[p + "res_k"] = cache.residual_keys()
        out[p + "res_v"] = cache.residual_values()
        if cache.s_state is not None:
            out[p + "s_state"] = cache.s_state
            out[p + "p_state"] = cache.p_state
        fp = memory_footprint(cache)
        out[p + "footprint"] = np.array([fp.packed_codes, fp.scales_zeros, fp.residual,
                                         fp.correction_states])
        out[p + "kvlc"] = np.frombuffer(serialize_cache(cache), np.uint8)
        # decode outputs: queries x block sizes x literal, with partials
        qs = rng(dseed + 1000).standard_normal((3, d))
        if name == "c_lit":
            qs = qs * 3
        out[p + "q"] = qs
        blocks = (None, 16, 32) if g >= 32 else (None, 4)
        for qi, q in enumerate(qs):
            for bi, blk in enumerate(blocks):
                for lit in (False, True):
                    if cache.tokens_total == 0:
                        continue
                    o, part = decode_step_blocked(q, cache, ad, block_tokens=blk,
                                                  literal_correction=lit,
                                                  return_partials=True)
                    key = f"{p}dec/{qi}_{bi}_{int(lit)}"
                    out[key + "/out"] = o
                    out[key + "/y"] = part.y_partial
                    out[key + "/m"] = part.block_max
                    out[key + "/l"] = part.block_sum
            if ad is not None:
                out[f"{p}dec/{qi}_noad/out"] = decode_step_blocked(q, cache, None)
        out[p + "blocks"] = np.array([-1 if b is None else b for b in blocks])
    # correction-dominated extreme logits (test_attention.py:267-277)
    d = 8
    ad = CorrectionAdapter.initialize(d, 8, seed=10)
    cache = KVCacheState(d, group_size=8, residual_window=0)
    gen = rng(15)
    vs = []
    for _ in range(16):
        v_t = gen.standard_normal(d)
        vs.append(v_t)
        cache.append(np.ones(d), v_t, ad)
    out["ext/v"] = np.asarray(vs)
    for sign in (300.0, -300.0):
        out[f"ext/out_{int(sign)}"] = decode_step_blocked(np.full(d, sign), cache, ad)
    return out


ATTN_CASES = [  # name, seed, n, d, rank (0 = no adapter), adapter seed
    ("a_small", 0, 24, 8, 8, 3),
    ("a_noad", 1, 40, 16, 0, 0),
    ("a_mid", 2, 96, 32, 16, 7),
    ("a_prod", 3, 300, 128, 256, 0),
]


def attention_cases():
    """Causal prefill attention (attention.py:50-155) on quantized inputs built like the
    reference tests' quantized_inputs (test_attention.py:145-154)."""
    out = {}
    for name, seed, n, d, rank, aseed in ATTN_CASES:
        g = rng(seed)
        q = g.standard_normal((n, d))
        k = g.standard_normal((n, d))
        v = g.standard_normal((n, d))
        k_hat = quantize_tensor(k, QuantConfig(bits=2, group_size=n, axis="channel")).dequantize()
        v_hat = quantize_tensor(v, QuantConfig(bits=2, group_size=d, axis="token")).dequantize()
        ad = CorrectionAdapter.initialize(d, rank, seed=aseed) if rank else None
        p = f"{name}/"
        out[p + "meta"] = np.array([seed, n, d, rank, aseed])
        out[p + "q"], out[p + "k_hat"], out[p + "k_err"], out[p + "v_hat"] = q, k_hat, k - k_hat, v_hat
        w, y = attention_reference(q, k_hat, v_hat)
        out[p + "ref_w"], out[p + "ref_y"] = w, y
        cq, cr = OpCounter(), OpCounter()
        out[p + "quad"] = corrected_attention_quadratic(q, k_hat, k - k_hat, v_hat, ad, cq)
        out[p + "rec"] = corrected_attention_recurrent(q, k_hat, k - k_hat, v_hat, ad, cr)
        out[p + "macs"] = np.array([cq.macs, cr.macs])
    return out


def train_cases():
    """Adapter calibration (adapter.py:104-307): corrected rows, per-item and batched
    loss / gradients, a short Adam run, the .kvla bytes."""
    out = {}
    g = rng(90)
    n, d, rank = 48, 16, 8
    q = g.standard_normal((n, d))
    k = g.standard_normal((n, d))
    v = g.standard_normal((n, d))
    k_hat = quantize_tensor(k, QuantConfig(bits=2, group_size=16, axis="channel")).dequantize()
    k_err = k - k_hat
    ad = CorrectionAdapter.initialize(d, rank, seed=4)
    a_full, _ = attention_reference(q, k, v)
    out["t/q"], out["t/k"], out["t/v"], out["t/k_hat"] = q, k, v, k_hat
    out["t/cw"] = corrected_weights(q[10], k_hat[:11], k_err[:11], ad)
    batch = [(a_full[t, : t + 1], q[t], k_hat[: t + 1], k_err[: t + 1]) for t in (3, 17, 40)]
    loss, grads = loss_and_grads(batch, ad)
    out["t/item_loss"] = np.array([loss])
    for name, gr in grads.items():
        out[f"t/item_{name}"] = gr
    pos = np.array([2, 9, 30, 47])
    loss, grads = _batched_loss_and_grads(a_full, pos, q, k_hat, k_err, ad)
    out["t/batch_loss"] = np.array([loss])
    for name, gr in grads.items():
        out[f"t/batch_{name}"] = gr
    trained, losses = train_adapter(q, k, v, TrainSettings(rank=rank, steps=6, lr=0.05, batch=16, seed=2,
                                                           group_size=16))
    out["t/losses"] = np.asarray(losses)
    for name in ("w1_q", "w2_q", "w1_k", "w2_k"):
        out[f"t/trained_{name}"] = getattr(trained, name)
    out["t/kvla"] = np.frombuffer(serialize_adapter(ad), np.uint8)
    return out


def main():
    for fname, fn in (("quantize", quantize_cases), ("hadamard", hadamard_cases),
                      ("adapter", adapter_cases), ("cache", cache_cases), ("attention", attention_cases), ("train", train_cases)):
        data = fn()
        path = os.path.join(HERE, f"{fname}.npz")
        np.savez_compressed(path, **data)
        print(f"wrote {path}: {len(data)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
