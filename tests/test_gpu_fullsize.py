"""Parity at the BASELINE sizes (configs 2, 3 and 4) on sampled units.

The whole batch is prefilled and decoded on the GPU at full size; a seeded
sample of (b, kv-head) units is rebuilt by the oracle (a unit is independent of
the others) and compared: T1 code words and T2 fp16 metadata of
sampled chunks bit-exact, T3 S / P, T4 decode output of the unit's query heads.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
from kvlc_testutil import bf16_round  # noqa: E402

D = 128


def _bf16(shape, g):
    return torch.from_numpy(g.standard_normal(shape).astype(np.float32)).bfloat16()


def _check_units(cache, k, v, q, units, bank_seeds, chunk_sample, s_tol=1e-5, out_tol=1e-3):
    Hkv, Hq = cache.Hkv, cache.Hq
    NG = Hq // Hkv
    out = cache.decode(q.cuda(), adapters=AdapterBank.initialize(Hkv, seeds=bank_seeds), out_dtype=torch.float32)
    out = out.cpu().numpy()
    qn = q.float().numpy().astype(np.float64)
    for (b, h) in units:
        ad = orc.init_adapter(D, 256, seed=bank_seeds[h])
        kk = k[b, h].float().numpy().astype(np.float64)
        vv = v[b, h].float().numpy().astype(np.float64)
        oc = orc.build_cache(kk, vv, ad)
        assert cache.n_chunks[b] == len(oc.key_chunks)
        for ci in chunk_sample(len(oc.key_chunks)):
            ex = cache.export_chunk(b, h, ci)
            ch = oc.key_chunks[ci]
            assert np.array_equal(ex["kwords"], ch.words), (b, h, ci)
            assert np.array_equal(ex["kscale"], ch.scales[0].astype(np.float16)), (b, h, ci)
            sl = slice(ci * 128, (ci + 1) * 128)
            assert np.array_equal(ex["vwords"], oc.value_words[sl]), (b, h, ci)
            assert np.array_equal(ex["vzero"], oc.value_zeros[sl, 0].astype(np.float16)), (b, h, ci)
        u = b * Hkv + h
        S = cache.S[u].double().cpu().numpy()
        assert np.linalg.norm(S - oc.s_state) <= s_tol * np.linalg.norm(oc.s_state), (b, h)
        ocm = orc.fp16_meta_copy(oc)
        for i in range(NG):
            ref = orc.decode_blocked(qn[b, h * NG + i], ocm, ad)
            err = np.abs(out[b, h * NG + i] - ref).max()
            assert err <= out_tol * np.abs(ref).max(), (b, h, i, err)


@pytest.mark.parametrize("cfg", ["config2", "config3"])
def test_full_batch_8k_sampled_units(cfg):
    B, Hkv, Hq, n = (16, 8, 32, 8192) if cfg == "config2" else (16, 4, 28, 8192)
    g = orc.rng(2024 if cfg == "config2" else 2025)
    k, v, q = _bf16((B, Hkv, n, D), g), _bf16((B, Hkv, n, D), g), _bf16((B, Hq, D), g)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    seeds = list(range(Hkv))
    cache.prefill(k.cuda(), v.cuda(), adapters=AdapterBank.initialize(Hkv, seeds=seeds))
    units = [(0, 0), (7, Hkv - 1), (15, Hkv // 2)]
    _check_units(cache, k, v, q, units, seeds, lambda nc: [0, nc // 2, nc - 1])


def test_config4_128k_one_sequence_sampled_unit():
    B, Hkv, Hq, n = 1, 8, 32, 131072
    g = orc.rng(2026)
    k, v, q = _bf16((B, Hkv, n, D), g), _bf16((B, Hkv, n, D), g), _bf16((B, Hq, D), g)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    seeds = list(range(Hkv))
    cache.prefill(k.cuda(), v.cuda(), adapters=AdapterBank.initialize(Hkv, seeds=seeds))
    assert int(cache.n_chunks[0]) == (n - 128) // 128
    # T3 / T4 stated for a 131k-token state: the fp32 tensor-core accumulation
    # of S measures 1.9e-5 relative (4.5e-6 at 8k, growing ~ sqrt(n)); the decode output, an
    # average over 131k values (max|out| ~ 0.016) against O(1) correction terms, carries that
    # state error as 1.4e-3 .. 2.0e-3 of max|out| (north_star's stated example: 1e-2)
    _check_units(cache, k, v, q, [(0, 3)], seeds, lambda nc: [0, 511, nc - 1], s_tol=3e-5, out_tol=3e-3)
