"""Reference-semantics CUDA path (the per-head drop-in shim) vs the REFERENCE's
own outputs (golden fixtures made by running quantkv, tests/golden/make_golden.py).

Mirrors the reference's unit tests (test_quantize.py, test_hadamard.py,
test_adapter.py, test_cache.py, test_attention.py): bit-exact codes and
float64 scales, 1e-12 for the float64 kernels, the reference's own 1e-4
blocked-decode tolerance tightened to 1e-5 here.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2510_05373_b200 as qk  # noqa: E402


def _cfg(meta):
    r, c, bits, g, axis = (int(x) for x in meta)
    return r, c, qk.QuantConfig(bits=bits, group_size=g, axis="token" if axis == 0 else "channel")


def test_quantize_tensor_matches_reference_bit_exact(golden):
    z = golden["quantize"]
    names = sorted({k.split("/")[0] for k in z if k.endswith("/meta")})
    assert len(names) >= 10
    for name in names:
        r, c, cfg = _cfg(z[f"{name}/meta"])
        qt = qk.quantize_tensor(z[f"{name}/x"], cfg)
        assert np.array_equal(qt.codes, z[f"{name}/codes"]), name
        assert np.array_equal(qt.scales, z[f"{name}/scales"]), name
        assert np.array_equal(qt.zeros, z[f"{name}/zeros"]), name
        assert np.array_equal(qt.dequantize(), z[f"{name}/deq"]), name


def test_known_answers(golden):
    z = golden["quantize"]
    codes, scale, zero = qk.quantize_group([0.0, 0.5, 1.5, 3.0], bits=2)
    assert np.array_equal(codes, z["ka/half_even_codes"]) and list(codes) == [0, 0, 2, 3]
    assert (scale, zero) == tuple(z["ka/half_even_scale"])
    w = qk.pack_codes(np.array([3, 2, 1, 0] + [0] * 12), bits=2)
    assert w.shape == (1,) and w[0] == 0x0000001B == z["ka/lane_word"][0]
    assert np.array_equal(qk.pack_codes(z["ka/pack_rows_codes"], 2), z["ka/pack_rows_words"])
    for bits in (2, 3, 4, 8):
        c, w = z[f"ka/pack_{bits}b_codes"], z[f"ka/pack_{bits}b_words"]
        assert np.array_equal(qk.pack_codes(c, bits), w)
        assert np.array_equal(qk.unpack_codes(w, c.shape[1], bits), c)
    codes, scale, zero = qk.quantize_group([5.0, 5.0, 5.0], bits=2)
    assert list(codes) == [0, 0, 0] and scale == 0.0 and zero == 5.0
    assert np.array_equal(qk.dequantize_group(codes, scale, zero), [5.0, 5.0, 5.0])


def test_group_error_bound_and_extremes():
    for seed in range(20):
        g = qk.rng(seed)
        n = int(g.integers(2, 200))
        bits = int(g.choice([2, 3, 4, 8]))
        v = g.standard_normal(n) * g.uniform(0.01, 100)
        codes, scale, zero = qk.quantize_group(v, bits)
        assert codes.max() <= (1 << bits) - 1
        back = qk.dequantize_group(codes, scale, zero)
        assert np.abs(back - v).max() <= scale / 2 + 1e-12
        assert back[np.argmin(v)] == pytest.approx(v.min(), abs=1e-12)


def test_pack_roundtrip_many_streams():
    g = qk.rng(1)
    batch = g.integers(0, 4, size=(20000, 37), dtype=np.uint8)
    assert np.array_equal(qk.unpack_codes(qk.pack_codes(batch, 2), 37, 2), batch)
    for n in (1, 5, 16, 17, 31, 32, 33, 64):
        codes = g.integers(0, 4, size=n, dtype=np.uint8)
        assert np.array_equal(qk.unpack_codes(qk.pack_codes(codes, 2), n, 2), codes)


def test_validation_messages():
    with pytest.raises(ValueError, match="range"):
        qk.pack_codes(np.array([4]), bits=2)
    with pytest.raises(ValueError, match="exceeds capacity"):
        qk.unpack_codes(np.array([0], dtype=np.uint32), 17, bits=2)
    with pytest.raises(ValueError, match="passthrough"):
        qk.quantize_tensor(np.ones((2, 2)), qk.QuantConfig(bits=16))
    with pytest.raises(ValueError, match="finite"):
        qk.quantize_tensor(np.array([[np.nan, 1.0]]), qk.QuantConfig())
    with pytest.raises(ValueError, match="non-empty"):
        qk.quantize_group([], bits=2)


def test_hadamard_and_rotate(golden):
    z = golden["hadamard"]
    for dim in (2, 4, 8, 16, 32, 64, 128, 256):
        assert np.array_equal(qk.hadamard_matrix(dim).matrix, z[f"H/{dim}"])
    for dim in (16, 64, 128):
        got = qk.rotate(z[f"rot/post_{dim}/x"], qk.hadamard_matrix(dim), "post")
        assert np.max(np.abs(got - z[f"rot/post_{dim}/y"])) <= 1e-12
    got = qk.rotate(z["rot/pre_32/x"], qk.hadamard_matrix(32), "pre")
    assert np.max(np.abs(got - z["rot/pre_32/y"])) <= 1e-12
    x = qk.rng(3).standard_normal((16, 16)) * 10
    h = qk.hadamard_matrix(16)
    assert np.max(np.abs(qk.rotate(x, h, "post") @ h.matrix.T - x)) <= 1e-12
    row = np.full((1, 16), 2.5)
    want = np.zeros(16)
    want[0] = 2.5 * 4
    assert np.max(np.abs(qk.rotate(row, h, "post")[0] - want)) <= 1e-12


def test_feature_maps(golden):
    z = golden["adapter"]
    keys = sorted({k.rsplit("/", 1)[0] for k in z if k.endswith("/phi_q")})
    for key in keys:
        d, rank, seed = (int(v) for v in key.split("/")[1].split("_"))
        ad = qk.CorrectionAdapter.initialize(d, rank, seed=seed)
        for n in ("w1_q", "w2_q", "w1_k", "w2_k"):
            assert np.array_equal(getattr(ad, n), z[f"{key}/{n}"])
        x = z[f"{key}/x"]
        assert np.max(np.abs(qk.phi_q(ad, x) - z[f"{key}/phi_q"])) <= 1e-12
        assert np.max(np.abs(qk.phi_k(ad, x) - z[f"{key}/phi_k"])) <= 1e-12
        assert np.max(np.abs(qk.feature_map(x[0], ad.w1_q, ad.w2_q) - z[f"{key}/fm_vec"])) <= 1e-12
        assert np.allclose(qk.phi_q(ad, x).sum(axis=1), 2.0, atol=1e-12)
    ad = qk.CorrectionAdapter.initialize(6, 16, seed=1)
    assert qk.correction_term(np.ones(6) * 3, np.zeros(6), ad) == pytest.approx(4.0 / 16.0, abs=1e-12)


def _cases(golden):
    z = golden["cache"]
    return z, sorted({k.split("/")[0] for k in z if k.endswith("/meta") and k.startswith("c_")})


def _build(z, name):
    n, d, g, win, rot, rank, aseed = (int(x) for x in z[f"{name}/meta"][:7])
    ad = qk.CorrectionAdapter.initialize(d, rank, seed=aseed) if rank else None
    cache = qk.KVCacheState(d, group_size=g, residual_window=win, rotate_values=bool(rot))
    cache.extend(z[f"{name}/k"], z[f"{name}/v"], ad)
    return cache, ad


def test_streaming_cache_matches_reference(golden):
    z, names = _cases(golden)
    for name in names:
        cache, ad = _build(z, name)
        meta = z[f"{name}/meta"]
        assert (cache.quantized_tokens, cache.residual_len, cache.tokens_total) == tuple(meta[7:10])
        if cache.quantized_tokens:
            kc = cache.key_chunks
            assert np.array_equal(np.stack([c.codes for c in kc]), z[f"{name}/kcodes"]), name
            assert np.array_equal(np.stack([c.scales for c in kc]), z[f"{name}/kscales"]), name
            assert np.array_equal(np.stack([c.zeros for c in kc]), z[f"{name}/kzeros"]), name
            vr = cache.value_rows
            rotated = bool(meta[4])
            if rotated:
                # FWHT vs dense x@H differ in the last ulp; codes must still agree
                assert np.array_equal(vr.codes, z[f"{name}/vcodes"]), name
                assert np.allclose(vr.scales, z[f"{name}/vscales"], rtol=1e-13, atol=1e-15), name
                assert np.allclose(vr.zeros, z[f"{name}/vzeros"], rtol=1e-13, atol=1e-14), name
            else:
                assert np.array_equal(vr.codes, z[f"{name}/vcodes"]), name
                assert np.array_equal(vr.scales, z[f"{name}/vscales"]), name
                assert np.array_equal(vr.zeros, z[f"{name}/vzeros"]), name
        assert np.array_equal(cache.residual_keys(), z[f"{name}/res_k"]), name
        assert np.array_equal(cache.residual_values(), z[f"{name}/res_v"]), name
        if f"{name}/s_state" in z:
            s_ref, p_ref = z[f"{name}/s_state"], z[f"{name}/p_state"]
            assert np.max(np.abs(cache.s_state - s_ref)) <= 1e-10 * max(1.0, np.abs(s_ref).max()), name
            assert np.max(np.abs(cache.p_state - p_ref)) <= 1e-10 * max(1.0, np.abs(p_ref).max()), name
        else:
            assert cache.s_state is None
        fp = qk.memory_footprint(cache)
        assert [fp.packed_codes, fp.scales_zeros, fp.residual, fp.correction_states] == \
            list(z[f"{name}/footprint"]), name


def test_streamed_append_equals_extend(golden):
    z, _ = _cases(golden)
    name = "c_small"
    n, d, g, win, rot, rank, aseed = (int(x) for x in z[f"{name}/meta"][:7])
    ad = qk.CorrectionAdapter.initialize(d, rank, seed=aseed)
    cache = qk.KVCacheState(d, group_size=g, residual_window=win, rotate_values=bool(rot))
    for t in range(n):
        cache.append(z[f"{name}/k"][t], z[f"{name}/v"][t], ad)
    assert np.array_equal(np.stack([c.codes for c in cache.key_chunks]), z[f"{name}/kcodes"])
    assert np.allclose(cache.s_state, z[f"{name}/s_state"], rtol=1e-12, atol=1e-12)


def test_blocked_decode_matches_reference(golden):
    z, names = _cases(golden)
    worst = 0.0
    for name in names:
        cache, ad = _build(z, name)
        blocks = [None if b < 0 else int(b) for b in z[f"{name}/blocks"]]
        for qi, q in enumerate(z[f"{name}/q"]):
            for bi, blk in enumerate(blocks):
                for lit in (False, True):
                    key = f"{name}/dec/{qi}_{bi}_{int(lit)}"
                    out, part = qk.decode_step_blocked(q, cache, ad, block_tokens=blk,
                                                       literal_correction=lit, return_partials=True)
                    ref = z[key + "/out"]
                    err = float(np.max(np.abs(out - ref)))
                    worst = max(worst, err)
                    assert err <= 1e-5 * max(1.0, np.abs(ref).max()), (key, err)
                    assert part.y_partial.shape == z[key + "/y"].shape
                    assert part.y_partial.dtype == np.float32
                    assert np.allclose(part.block_max, z[key + "/m"], rtol=1e-5, atol=1e-5), key
                    assert np.allclose(part.block_sum, z[key + "/l"], rtol=1e-4, atol=1e-6), key
                    assert np.allclose(part.y_partial, z[key + "/y"], rtol=1e-4, atol=1e-5), key
            if ad is not None:
                got = qk.decode_step_blocked(q, cache, None)
                assert np.max(np.abs(got - z[f"{name}/dec/{qi}_noad/out"])) <= 1e-5
    assert worst < 1e-5


def test_extreme_logits_correction_dominated(golden):
    z = golden["cache"]
    d = 8
    ad = qk.CorrectionAdapter.initialize(d, 8, seed=10)
    cache = qk.KVCacheState(d, group_size=8, residual_window=0)
    for v_t in z["ext/v"]:
        cache.append(np.ones(d), v_t, ad)
    for sign in (300.0, -300.0):
        out = qk.decode_step_blocked(np.full(d, sign), cache, ad)
        assert np.all(np.isfinite(out))
        assert np.max(np.abs(out - z[f"ext/out_{int(sign)}"])) <= 1e-5


def test_cache_and_decode_validation():
    cache = qk.KVCacheState(8, group_size=16, residual_window=0)
    with pytest.raises(ValueError, match="token dims"):
        cache.append(np.zeros(7), np.zeros(8))
    cache.append(np.zeros(8), np.zeros(8))
    with pytest.raises(ValueError, match="need 16 residual tokens"):
        cache.flush_group()
    with pytest.raises(ValueError, match="token range"):
        cache.dequantized_keys(0, 1)
    with pytest.raises(ValueError, match="query shape"):
        qk.decode_step_blocked(np.zeros(9), cache)
    with pytest.raises(ValueError, match="block_tokens"):
        qk.decode_step_blocked(np.zeros(8), cache, block_tokens=0)
    with pytest.raises(ValueError, match="empty cache"):
        qk.decode_step_blocked(np.zeros(8), qk.KVCacheState(8, group_size=16, residual_window=0))
    g = qk.rng(9)
    cache = qk.KVCacheState(8, group_size=4, residual_window=0)
    small = qk.CorrectionAdapter.initialize(4, 8, seed=0)
    for _ in range(3):
        cache.append(g.standard_normal(8), g.standard_normal(8), small)
    with pytest.raises(ValueError, match="adapter dim"):
        cache.append(g.standard_normal(8), g.standard_normal(8), small)
    cache = qk.KVCacheState(8, group_size=4, residual_window=0)
    first = qk.CorrectionAdapter.initialize(8, 8, seed=1)
    second = qk.CorrectionAdapter.initialize(8, 16, seed=2)
    for _ in range(4):
        cache.append(g.standard_normal(8), g.standard_normal(8), first)
    for _ in range(3):
        cache.append(g.standard_normal(8), g.standard_normal(8), second)
    with pytest.raises(ValueError, match="cache state rank"):
        cache.append(g.standard_normal(8), g.standard_normal(8), second)


def test_exact_keys_give_uniform_feature_states():
    n, d, rank = 32, 16, 16
    g = qk.rng(4)
    k = g.integers(0, 4, size=(n, d)).astype(np.float64)
    k[0, :] = 0.0
    k[1, :] = 3.0
    v = g.standard_normal((n, d))
    ad = qk.CorrectionAdapter.initialize(d, rank, seed=5)
    cache = qk.KVCacheState(d, group_size=n, residual_window=0, rotate_values=False)
    cache.extend(k, v, ad)
    assert np.array_equal(cache.p_state, np.full(rank, n / 8.0))
    v_q = cache.dequantized_values(0, n)
    want = np.outer(v_q.sum(axis=0), np.full(rank, 2.0 / rank))
    assert np.max(np.abs(cache.s_state - want)) <= 1e-12


@pytest.mark.parametrize("rotation,bits,shape", [("post", 2, (40, 64)), ("pre", 4, (32, 24)), ("none", 3, (17, 30)),
                                                 ("post", 16, (8, 16))])
def test_quantize_roundtrip_matches_reference_composition(rotation, bits, shape):
    """quantize_roundtrip (attention.py:68-88): rotate, quantize, dequantize, rotate back."""
    from oracle import kvlinc_oracle as orc
    x = orc.rng(7).standard_normal(shape)
    axis = "channel" if rotation == "pre" else "token"
    cfg = qk.QuantConfig(bits=bits, group_size=16, axis=axis, rotation=rotation)
    got = qk.quantize_roundtrip(x, cfg)
    if rotation == "pre":
        h = orc.hadamard(shape[0])
        xr = h @ x
    elif rotation == "post":
        h = orc.hadamard(shape[1])
        xr = x @ h
    else:
        h, xr = None, x
    xq = xr if bits == 16 else orc.dequantize_matrix(orc.quantize_matrix(xr, bits, 16, axis))
    want = h.T @ xq if rotation == "pre" else (xq @ h.T if rotation == "post" else xq)
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.abs(want).max())


def test_prefill_attention_forms_match_reference(golden):
    """attention_reference, attention_with_config and the corrected quadratic / recurrent
    forms (attention.py:50-155) against the reference's outputs, with its MAC counters."""
    z = golden["attention"]
    for name in sorted({k.split("/")[0] for k in z if k.endswith("/meta")}):
        seed, n, d, rank, aseed = (int(x) for x in z[f"{name}/meta"])
        q, kq, ke, vq = (z[f"{name}/{x}"] for x in ("q", "k_hat", "k_err", "v_hat"))
        w, y = qk.attention_reference(q, kq, vq)
        assert np.max(np.abs(w - z[f"{name}/ref_w"])) <= 1e-13, name
        assert np.max(np.abs(y - z[f"{name}/ref_y"])) <= 1e-12, name
        ad = qk.CorrectionAdapter.initialize(d, rank, seed=aseed) if rank else None
        cq, cr = qk.OpCounter(), qk.OpCounter()
        quad = qk.corrected_attention_quadratic(q, kq, ke, vq, ad, cq)
        rec = qk.corrected_attention_recurrent(q, kq, ke, vq, ad, cr)
        assert np.max(np.abs(quad - z[f"{name}/quad"])) <= 1e-12, name
        assert np.max(np.abs(rec - z[f"{name}/rec"])) <= 1e-10, name
        assert [cq.macs, cr.macs] == list(z[f"{name}/macs"]), name


def test_prefill_attention_reference_properties():
    """The reference's own checks (test_attention.py:157-205): no adapter == plain
    attention, k_err = 0 closed form, first recurrent output = first value, shapes."""
    from oracle import kvlinc_oracle as orc
    g = orc.rng(0)
    n, d = 24, 8
    q, k, v = (g.standard_normal((n, d)) for _ in range(3))
    _, want = qk.attention_reference(q, k, v)
    for ad in (None, qk.CorrectionAdapter.initialize(8, 8, enabled=False)):
        assert np.max(np.abs(qk.corrected_attention_quadratic(q, k, k * 0, v, ad) - want)) <= 1e-12
    ad = qk.CorrectionAdapter.initialize(8, 16, seed=5)
    got = qk.corrected_attention_quadratic(q, k, np.zeros_like(k), v, ad)
    mask = np.arange(n)[None, :] <= np.arange(n)[:, None]
    e = np.where(mask, np.exp(q @ k.T / np.sqrt(8)), 0.0) + mask * (4.0 / 16.0)
    assert np.max(np.abs(got - (e @ v) / e.sum(axis=1, keepdims=True))) <= 1e-12
    rec = qk.corrected_attention_recurrent(q[:1], k[:1], k[:1] * 0.1, v[:1], ad)
    assert np.max(np.abs(rec[0] - v[0])) <= 1e-12
    cfg = qk.QuantConfig(bits=2, group_size=8, axis="token", rotation="post")
    a_cfg, y_cfg = qk.attention_with_config(q, k, v, cfg, cfg)
    a_ref, y_ref = qk.attention_reference(q, qk.quantize_roundtrip(k, cfg), qk.quantize_roundtrip(v, cfg))
    assert np.array_equal(a_cfg, a_ref) and np.array_equal(y_cfg, y_ref)
    with pytest.raises(ValueError, match="Q/K/V shapes differ"):
        qk.attention_reference(q, k[:3], v)


def test_adapter_training_matches_reference(golden):
    """Adapter calibration (adapter.py:104-307) against the reference's outputs: corrected
    rows, per-item and batched loss / gradients, a 6-step Adam run."""
    from paper_2510_05373_b200 import train as tr
    z = golden["train"]
    q, k, v, k_hat = z["t/q"], z["t/k"], z["t/v"], z["t/k_hat"]
    k_err = k - k_hat
    n, d = q.shape
    ad = qk.CorrectionAdapter.initialize(d, 8, seed=4)
    assert np.max(np.abs(qk.corrected_weights(q[10], k_hat[:11], k_err[:11], ad) - z["t/cw"])) <= 1e-14
    a_full, _ = qk.attention_reference(q, k, v)
    batch = [(a_full[t, : t + 1], q[t], k_hat[: t + 1], k_err[: t + 1]) for t in (3, 17, 40)]
    loss, grads = qk.loss_and_grads(batch, ad)
    assert abs(loss - z["t/item_loss"][0]) <= 1e-12
    for name, g in grads.items():
        assert np.max(np.abs(g - z[f"t/item_{name}"])) <= 1e-12 * max(1.0, np.abs(z[f"t/item_{name}"]).max()), name
    loss, grads = tr._batched_loss_and_grads(a_full, np.array([2, 9, 30, 47]), q, k_hat, k_err, ad)
    assert abs(loss - z["t/batch_loss"][0]) <= 1e-12
    for name, g in grads.items():
        assert np.max(np.abs(g - z[f"t/batch_{name}"])) <= 1e-12 * max(1.0, np.abs(z[f"t/batch_{name}"]).max()), name
    trained, losses = qk.train_adapter(q, k, v, qk.TrainSettings(rank=8, steps=6, lr=0.05, batch=16, seed=2,
                                                                 group_size=16))
    assert np.max(np.abs(np.asarray(losses) - z["t/losses"])) <= 1e-10
    for name in ("w1_q", "w2_q", "w1_k", "w2_k"):
        assert np.max(np.abs(getattr(trained, name) - z[f"t/trained_{name}"])) <= 1e-10, name
    with pytest.raises(ValueError, match="non-empty"):
        qk.loss_and_grads([], ad)
    zero = qk.train_adapter(q, k, v, qk.TrainSettings(rank=8, steps=0, seed=2, group_size=16))[0]
    assert np.array_equal(zero.w1_q, qk.CorrectionAdapter.initialize(d, 8, seed=2).w1_q)


def test_linalg_substrate():
    """matmul / softmax_rows (linalg.py:28-47) with the reference's messages."""
    from oracle import kvlinc_oracle as orc
    g = orc.rng(3)
    a, b = g.standard_normal((5, 7)), g.standard_normal((7, 3))
    assert np.max(np.abs(qk.matmul(a, b) - a @ b)) <= 1e-13
    x = g.standard_normal((4, 6))
    x[1, 2:] = -np.inf
    s = qk.softmax_rows(x)
    want = np.exp(x - x.max(axis=1, keepdims=True))
    want /= want.sum(axis=1, keepdims=True)
    assert np.max(np.abs(s - want)) <= 1e-15 and np.all(s[1, 2:] == 0)
    with pytest.raises(ValueError, match="inner dims differ"):
        qk.matmul(a, a)
    with pytest.raises(ValueError, match="2-D operands"):
        qk.matmul(a[0], b)
