""".kvlc export / import (serialize_cache / deserialize_cache, cache.py:197-307).

Against the REFERENCE's own bytes (tests/golden/cache.npz `*/kvlc`, written by
quantkv.serialize_cache): header, code words, f16 metadata and f16 residual
byte-identical; f16 S / P within one f16 ulp plus 1e-5 of the state's scale (the
serving cache accumulates S / P in fp32 with tensor cores, the reference in fp64 — T3).  Import -> export is the
identity; decode on an imported cache matches the oracle decode of the same
file (T4).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2510_05373_b200 as qk  # noqa: E402
from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200 import kvlc_format as fmt  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
from kvlc_testutil import bf16_round  # noqa: E402

D = 128


def assert_kvlc_equal(got: bytes, want: bytes, state_ulps: int = 1):
    hg, hw = fmt.parse_header(got), fmt.parse_header(want)
    assert hg == hw
    sg, sw = fmt.split(got, hg), fmt.split(want, hw)
    for name in sg:
        if name in ("s", "p"):
            # one f16 rounding apart, plus the T3 budget (1e-5 of the state's scale) that the
            # fp32 tensor-core accumulation may spend on near-zero entries
            a, b = sg[name].astype(np.float64), sw[name].astype(np.float64)
            tol = state_ulps * 2.0 ** -10 * np.abs(b) + (1e-5 * np.abs(b).max() if state_ulps else 0.0)
            assert np.all(np.abs(a - b) <= tol), (name, np.max(np.abs(a - b) - tol))
        else:
            assert np.array_equal(sg[name], sw[name]), name


def _prod_case(golden):
    z = golden["cache"]
    n, d, g, win, rot, rank, aseed = (int(x) for x in z["c_prod/meta"][:7])
    assert (d, g, win, rot, rank) == (128, 128, 128, 1, 256)
    return z, n, aseed


def test_batched_export_matches_reference_bytes(golden):
    z, n, aseed = _prod_case(golden)
    k = torch.from_numpy(z["c_prod/k"].astype(np.float32)).bfloat16().view(1, 1, n, D)
    v = torch.from_numpy(z["c_prod/v"].astype(np.float32)).bfloat16().view(1, 1, n, D)
    cache = BatchedKVCache(1, 1, 4, n + 256)
    cache.prefill(k, v, adapters=AdapterBank.initialize(1, seeds=[aseed]))
    assert_kvlc_equal(cache.serialize(0, 0), z["c_prod/kvlc"].tobytes())


def test_batched_export_ragged_matches_oracle_and_round_trips():
    """B=3 x Hkv=2 ragged (short / no-flush / long), adapters on; streaming appends
    after prefill move the ring start, so export must unwrap the residual ring."""
    B, Hkv, lens = 3, 2, [600, 200, 300]  # odd flush counts: ring start at slot 128
    g = orc.rng(31)
    n = max(lens) + 40
    k = bf16_round(g.standard_normal((B, Hkv, n, D)).astype(np.float32))
    v = bf16_round(g.standard_normal((B, Hkv, n, D)).astype(np.float32))
    bank = AdapterBank.initialize(Hkv)
    oads = [orc.init_adapter(D, 256, seed=h) for h in range(Hkv)]
    cache = BatchedKVCache(B, Hkv, 4 * Hkv, n + 256)
    kt, vt = torch.from_numpy(k.astype(np.float32)).bfloat16(), torch.from_numpy(v.astype(np.float32)).bfloat16()
    cache.prefill(kt[:, :, : min(lens)], vt[:, :, : min(lens)], adapters=bank)
    for i in range(min(lens), max(lens)):  # streaming tail
        act = np.array([i < L for L in lens])
        cache.append(kt[:, :, i].cuda(), vt[:, :, i].cuda(), adapters=bank, active=act)
    assert cache.res_start.any()
    fresh = BatchedKVCache(B, Hkv, 4 * Hkv, n + 256)
    for b in range(B):
        imgs = [cache.serialize(b, h) for h in range(Hkv)]
        for h in range(Hkv):
            oc = orc.build_cache(k[b, h, : lens[b]], v[b, h, : lens[b]], oads[h])
            assert_kvlc_equal(imgs[h], orc.serialize(oc))
        fresh.load(b, imgs)
        for h in range(Hkv):
            assert fresh.serialize(b, h) == imgs[h]
    assert np.array_equal(fresh.n_chunks, cache.n_chunks) and np.array_equal(fresh.res_len, cache.res_len)
    assert np.array_equal(fresh.state_rank, [256, 0, 256])
    # decode on the imported cache == oracle decode on the deserialized file (T4)
    q = bf16_round(g.standard_normal((B, 4 * Hkv, D)).astype(np.float32))
    out = fresh.decode(torch.from_numpy(q.astype(np.float32)).bfloat16().cuda(), adapters=bank,
                       out_dtype=torch.float32).cpu().numpy()
    for b in range(B):
        for hq in range(4 * Hkv):
            oc = orc.deserialize(fresh.serialize(b, hq // 4))
            ref = orc.decode_blocked(q[b, hq], oc, oads[hq // 4] if oc.rank else None)
            assert np.max(np.abs(out[b, hq] - ref)) <= 1e-3 * np.abs(ref).max(), (b, hq)


def test_batched_load_validates():
    cache = BatchedKVCache(1, 2, 8, 512)
    img = BatchedKVCache(1, 2, 8, 512)
    g = orc.rng(2)
    kv = torch.from_numpy(g.standard_normal((1, 2, 400, D)).astype(np.float32)).bfloat16()  # 2 chunks
    img.prefill(kv, kv)
    a, b = img.serialize(0, 0), img.serialize(0, 1)
    with pytest.raises(fmt.CacheFormatError, match="bad magic"):
        cache.load(0, [b"XXXX" + a[4:], b])
    with pytest.raises(fmt.CacheFormatError, match="trailing bytes"):
        cache.load(0, [a + b"\0", b])
    with pytest.raises(ValueError, match="one per kv head"):
        cache.load(0, [a])
    small = BatchedKVCache(1, 2, 8, 200)
    with pytest.raises(ValueError, match="exceeds capacity"):
        small.load(0, [a, b])
    other = qk.KVCacheState(64, group_size=32, residual_window=16)
    other.extend(np.ones((60, 64)), np.ones((60, 64)))
    with pytest.raises(ValueError, match="serving cache holds"):
        cache.load(0, [qk.serialize_cache(other)] * 2)


def test_shim_serialize_matches_reference_bytes(golden, tmp_path):
    """Per-head drop-in: serialize_cache / read_cache / write_cache, every golden case."""
    z = golden["cache"]
    names = sorted({key.split("/")[0] for key in z if key.endswith("/kvlc")})
    for name in names:
        n, d, g, win, rot, rank, aseed = (int(x) for x in z[f"{name}/meta"][:7])
        ad = qk.CorrectionAdapter.initialize(d, rank, seed=aseed) if rank else None
        cache = qk.KVCacheState(d, group_size=g, residual_window=win, rotate_values=bool(rot))
        cache.extend(z[f"{name}/k"], z[f"{name}/v"], ad)
        ref = z[f"{name}/kvlc"].tobytes()
        got = qk.serialize_cache(cache)
        assert_kvlc_equal(got, ref, state_ulps=0)
        path = tmp_path / f"{name}.kvlc"
        qk.write_cache(cache, path)
        back = qk.read_cache(path)
        assert qk.serialize_cache(back) == got, name
        assert (back.quantized_tokens, back.residual_len, back.adapter_rank) == \
            (cache.quantized_tokens, cache.residual_len, cache.adapter_rank)
        if back.quantized_tokens:
            q = orc.rng(5).standard_normal(d)
            oc = orc.deserialize(ref)
            oad = orc.init_adapter(d, rank, seed=aseed) if rank else None
            want = orc.decode_blocked(q, oc, oad)
            out = qk.decode_step_blocked(q, back, ad)
            assert np.max(np.abs(out - want)) <= 1e-5 * max(1.0, np.abs(want).max()), name
    with pytest.raises(qk.CacheFormatError, match="truncated"):
        qk.deserialize_cache(ref[:-3])
