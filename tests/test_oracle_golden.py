"""CPU: pin the oracle (oracle/kvlinc_oracle.py) to the REFERENCE's own outputs.

The golden fixtures were produced by running the reference package
(tests/golden/make_golden.py).  The oracle must reproduce codes, scales,
rotations and feature maps bit for bit, the streaming-cache states to float64
rounding and the blocked decode to float32 rounding; once pinned, the GPU
parity tests may use the oracle at shapes the fixtures do not cover.
"""
import numpy as np
import pytest

from oracle import kvlinc_oracle as orc


def test_quantize_matches_reference(golden):
    z = golden["quantize"]
    names = sorted({k.split("/")[0] for k in z if k.endswith("/meta")})
    for name in names:
        r, c, bits, g, axis = (int(v) for v in z[f"{name}/meta"])
        p = orc.quantize_matrix(z[f"{name}/x"], bits, g, "token" if axis == 0 else "channel")
        assert np.array_equal(p.words, z[f"{name}/codes"]), name
        assert np.array_equal(p.scales, z[f"{name}/scales"]), name
        assert np.array_equal(p.zeros, z[f"{name}/zeros"]), name
        assert np.array_equal(orc.dequantize_matrix(p), z[f"{name}/deq"]), name


def test_known_answers(golden):
    z = golden["quantize"]
    codes, scale, zero = orc.quantize_group([0.0, 0.5, 1.5, 3.0], 2)
    assert list(codes) == [0, 0, 2, 3] and (scale, zero) == tuple(z["ka/half_even_scale"])
    assert orc.pack(np.array([3, 2, 1, 0] + [0] * 12), 2)[0] == 0x0000001B == z["ka/lane_word"][0]
    assert np.array_equal(orc.pack(z["ka/pack_rows_codes"], 2), z["ka/pack_rows_words"])
    for bits in (2, 3, 4, 8):
        c, w = z[f"ka/pack_{bits}b_codes"], z[f"ka/pack_{bits}b_words"]
        assert np.array_equal(orc.pack(c, bits), w)
        assert np.array_equal(orc.unpack(w, c.shape[1], bits), c)
    codes, scale, zero = orc.quantize_group([5.0, 5.0, 5.0], 2)
    assert list(codes) == [0, 0, 0] and scale == 0.0 and zero == 5.0


def test_hadamard_and_rotation_bit_exact(golden):
    z = golden["hadamard"]
    for dim in (2, 4, 8, 16, 32, 64, 128, 256):
        assert np.array_equal(orc.hadamard(dim), z[f"H/{dim}"])
    for dim in (16, 64, 128):
        assert np.array_equal(orc.rotate_post(z[f"rot/post_{dim}/x"]), z[f"rot/post_{dim}/y"])
    assert np.array_equal(orc.rotate_pre(z["rot/pre_32/x"]), z["rot/pre_32/y"])


def test_feature_maps(golden):
    z = golden["adapter"]
    keys = sorted({k.rsplit("/", 1)[0] for k in z if k.endswith("/phi_q")})
    for key in keys:
        d, rank, seed = (int(v) for v in key.split("/")[1].split("_"))
        ad = orc.init_adapter(d, rank, seed=seed)
        for n in ("w1_q", "w2_q", "w1_k", "w2_k"):
            assert np.array_equal(getattr(ad, n), z[f"{key}/{n}"])
        assert np.max(np.abs(orc.phi_q(ad, z[f"{key}/x"]) - z[f"{key}/phi_q"])) <= 1e-15
        assert np.max(np.abs(orc.phi_k(ad, z[f"{key}/x"]) - z[f"{key}/phi_k"])) <= 1e-15


def _cache_cases(golden):
    z = golden["cache"]
    return z, sorted({k.split("/")[0] for k in z if k.endswith("/meta") and k.startswith("c_")})


def _build(z, name):
    n, d, g, win, rot, rank, aseed = (int(x) for x in z[f"{name}/meta"][:7])
    ad = orc.init_adapter(d, rank, seed=aseed) if rank else None
    return orc.build_cache(z[f"{name}/k"], z[f"{name}/v"], ad, group=g, window=win, rotate=bool(rot)), ad


def test_streaming_cache_matches_reference(golden):
    z, names = _cache_cases(golden)
    for name in names:
        c, _ = _build(z, name)
        meta = z[f"{name}/meta"]
        assert (c.quantized_tokens, c.residual_len, c.tokens_total) == tuple(meta[7:10])
        if c.quantized_tokens:
            assert np.array_equal(np.stack([k.words for k in c.key_chunks]), z[f"{name}/kcodes"])
            assert np.array_equal(np.stack([k.scales for k in c.key_chunks]), z[f"{name}/kscales"])
            assert np.array_equal(c.value_words, z[f"{name}/vcodes"]), name
            assert np.array_equal(c.value_scales, z[f"{name}/vscales"]), name
            assert np.array_equal(c.value_zeros, z[f"{name}/vzeros"]), name
        assert np.array_equal(c.residual_keys(), z[f"{name}/res_k"])
        if f"{name}/s_state" in z:
            assert np.array_equal(c.s_state, z[f"{name}/s_state"]), name
            assert np.array_equal(c.p_state, z[f"{name}/p_state"]), name
        fp = orc.footprint(c)
        assert [fp[k] for k in ("packed_codes", "scales_zeros", "residual", "correction_states")] == \
            list(z[f"{name}/footprint"])


def test_blocked_decode_matches_reference(golden):
    z, names = _cache_cases(golden)
    for name in names:
        c, ad = _build(z, name)
        blocks = [None if b < 0 else int(b) for b in z[f"{name}/blocks"]]
        for qi, q in enumerate(z[f"{name}/q"]):
            for bi, blk in enumerate(blocks):
                for lit in (False, True):
                    key = f"{name}/dec/{qi}_{bi}_{int(lit)}"
                    out, (y, m, l) = orc.decode_blocked(q, c, ad, block=blk, literal=lit,
                                                        return_partials=True)
                    assert np.max(np.abs(out - z[key + "/out"])) <= 1e-6, key
                    assert np.array_equal(m, z[key + "/m"]), key
                    assert np.allclose(y, z[key + "/y"], rtol=1e-6, atol=1e-7), key
                    assert np.allclose(l, z[key + "/l"], rtol=1e-6), key
            # the fp64 dense oracle agrees with the blocked path (acceptance c4 bound)
            assert np.max(np.abs(orc.decode_dense(q, c, ad) - z[f"{name}/dec/{qi}_0_0/out"])) <= 1e-4


def test_extreme_logits(golden):
    z = golden["cache"]
    ad = orc.init_adapter(8, 8, seed=10)
    c = orc.Cache(8, group=8, window=0, rotate=True)
    for v_t in z["ext/v"]:
        c.append(np.ones(8), v_t, ad)
    for sign in (300.0, -300.0):
        out = orc.decode_blocked(np.full(8, sign), c, ad)
        assert np.all(np.isfinite(out))
        assert np.max(np.abs(out - z[f"ext/out_{int(sign)}"])) <= 1e-6


def test_fp16_meta_copy_rounds_only_metadata(golden):
    z, _ = _cache_cases(golden)
    c, _ = _build(z, "c_rot")
    c16 = orc.fp16_meta_copy(c)
    assert np.array_equal(c16.value_words, c.value_words)
    assert np.array_equal(c16.value_scales, c.value_scales.astype(np.float16).astype(np.float64))
    assert c16.s_state is c.s_state or np.array_equal(c16.s_state, c.s_state)


@pytest.mark.parametrize("seed", [4100])
def test_value_rotation_tie_is_reference_ordered(seed):
    """A genuine (x-min)/scale = 0.5 +- 1ulp tie (found at n=4096, seed 4100,
    chunk 14, token 39, channel 17): the reference's dense x @ H decides code 1;
    the oracle must reproduce it (an FWHT in a different order gives 0)."""
    from kvlc_testutil import bf16_round
    g = orc.rng(seed)
    n = 4096
    bf16_round(g.standard_normal((1, 1, n, 128)).astype(np.float32))  # keys (same stream order)
    v = bf16_round(g.standard_normal((1, 1, n, 128)).astype(np.float32))[0, 0]
    blk = v[14 * 128:15 * 128]
    ref = blk @ orc.hadamard(128)          # numpy/OpenBLAS, as the reference computes it
    assert np.array_equal(orc.rotate_post(blk), ref)
    codes, s, zz = orc.quantize_rows(orc.rotate_post(blk), 2, 128)
    assert codes[39, 17] == 1


def test_serialization_matches_reference(golden):
    """.kvlc bytes (cache.py:197-307): the oracle writer reproduces the reference's
    serialize_cache output byte for byte; the reader round-trips it."""
    z, names = _cache_cases(golden)
    for name in names:
        c, _ = _build(z, name)
        ref = z[f"{name}/kvlc"].tobytes()
        assert orc.serialize(c) == ref, name
        assert orc.serialize(orc.deserialize(ref)) == ref, name


def test_prefill_attention_matches_reference(golden):
    """attention_reference and the corrected quadratic / recurrent forms (attention.py:50-155)."""
    z = golden["attention"]
    for name in sorted({k.split("/")[0] for k in z if k.endswith("/meta")}):
        seed, n, d, rank, aseed = (int(x) for x in z[f"{name}/meta"])
        q, kq, ke, vq = (z[f"{name}/{x}"] for x in ("q", "k_hat", "k_err", "v_hat"))
        w, y = orc.attention_reference(q, kq, vq)
        assert np.max(np.abs(w - z[f"{name}/ref_w"])) <= 1e-13, name
        assert np.max(np.abs(y - z[f"{name}/ref_y"])) <= 1e-12, name
        ad = orc.init_adapter(d, rank, seed=aseed) if rank else None
        c = orc.corrected_attention(q, kq, ke, vq, ad)
        assert np.max(np.abs(c - z[f"{name}/quad"])) <= 1e-12, name
        assert np.max(np.abs(c - z[f"{name}/rec"])) <= 1e-10, name
