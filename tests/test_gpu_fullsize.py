"""Parity at the BASELINE sizes (configs 2, 3 and 4) on sampled units, every chunk.

The whole batch is prefilled and decoded on the GPU at full size; a seeded
sample of (b, kv-head) units (8 per config, all 4 at B1 x 4k) is rebuilt by the
oracle in parallel host processes (a unit is independent of the others, SURVEY
§8e) and compared at the survey's bounds:
  T1  code words of EVERY chunk of each sampled unit bit-exact (reference layout),
  T2  fp16 key / value scale and zero of every chunk equal float16(fp64 value),
  T3  S and P within relative Frobenius 1e-5 of the fp64 reference,
  T4  decode output of the unit's query heads within 1e-3 * max|ref| of
      decode_step_blocked on the fp16-metadata reference cache.
Configs: 2 = Llama-3-8B B16 x 8k; 3 = Qwen2.5-7B (28 q / 4 kv heads) at B1 x 4k,
B16 x 8k and B64 x 32k (the largest single-GPU point of SURVEY §8(d)); 4 =
Llama-3-8B B1 x 128k (131072 tokens, 1023 chunks).
"""
import multiprocessing as mp

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402

D = 128
S_TOL, OUT_TOL = 1e-5, 1e-3  # T3, T4


def _bf16(shape, g):
    return torch.from_numpy(g.standard_normal(shape).astype(np.float32)).bfloat16()


def _oracle_unit(args):
    kk, vv, seed = args
    ad = orc.init_adapter(D, 256, seed=seed)
    return orc.build_cache(kk, vv, ad)


def _oracle_caches(k, v, units, seeds):
    jobs = [(k[b, h].float().numpy().astype(np.float64), v[b, h].float().numpy().astype(np.float64), seeds[h])
            for (b, h) in units]
    with mp.get_context("fork").Pool(min(len(jobs), max(1, mp.cpu_count()))) as pool:
        return pool.map(_oracle_unit, jobs)


def _check_units(cache, k, v, q, units, seeds):
    Hkv, Hq = cache.Hkv, cache.Hq
    NG = Hq // Hkv
    out = cache.decode(q.cuda(), adapters=AdapterBank.initialize(Hkv, seeds=seeds), out_dtype=torch.float32)
    out = out.cpu().numpy()
    qn = q.float().numpy().astype(np.float64)
    worst = {"S": 0.0, "P": 0.0, "out": 0.0}
    for (b, h), oc in zip(units, _oracle_caches(k, v, units, seeds)):
        n = len(oc.key_chunks)
        assert int(cache.n_chunks[b]) == n
        ex = cache.export_unit(b, h, n)
        for ci in range(n):  # T1 / T2 on every chunk
            ch = oc.key_chunks[ci]
            sl = slice(ci * 128, (ci + 1) * 128)
            assert np.array_equal(ex["kwords"][ci], ch.words), (b, h, ci)
            assert np.array_equal(ex["kscale"][ci], ch.scales[0].astype(np.float16)), (b, h, ci)
            assert np.array_equal(ex["kzero"][ci], ch.zeros[0].astype(np.float16)), (b, h, ci)
            assert np.array_equal(ex["vwords"][ci], oc.value_words[sl]), (b, h, ci)
            assert np.array_equal(ex["vscale"][ci], oc.value_scales[sl, 0].astype(np.float16)), (b, h, ci)
            assert np.array_equal(ex["vzero"][ci], oc.value_zeros[sl, 0].astype(np.float16)), (b, h, ci)
        u = b * Hkv + h
        S = cache.S[u].double().cpu().numpy()
        P = cache.P[u].double().cpu().numpy()
        es = np.linalg.norm(S - oc.s_state) / np.linalg.norm(oc.s_state)
        ep = np.linalg.norm(P - oc.p_state) / np.linalg.norm(oc.p_state)
        assert es <= S_TOL and ep <= S_TOL, (b, h, es, ep)
        ad = orc.init_adapter(D, 256, seed=seeds[h])
        ocm = orc.fp16_meta_copy(oc)
        for i in range(NG):
            ref = orc.decode_blocked(qn[b, h * NG + i], ocm, ad)
            err = np.abs(out[b, h * NG + i] - ref).max() / np.abs(ref).max()
            assert err <= OUT_TOL, (b, h, i, err)
            worst["out"] = max(worst["out"], err)
        worst["S"], worst["P"] = max(worst["S"], es), max(worst["P"], ep)
    print("worst", {k2: f"{v2:.2e}" for k2, v2 in worst.items()})


def _sample_units(B, Hkv, n_units, seed):
    if B * Hkv <= n_units:
        return [(b, h) for b in range(B) for h in range(Hkv)]
    r = np.random.default_rng(seed)
    picks = r.choice(B * Hkv, size=n_units, replace=False)
    # always include the first and the last unit
    picks[0], picks[-1] = 0, B * Hkv - 1
    return [(int(p) // Hkv, int(p) % Hkv) for p in sorted(set(int(x) for x in picks))]


CONFIGS = {
    "config2_b16_8k": (16, 8, 32, 8192, 2024),
    "config3_b1_4k": (1, 4, 28, 4096, 2027),
    "config3_b16_8k": (16, 4, 28, 8192, 2025),
    "config3_b64_32k": (64, 4, 28, 32768, 2028),
    "config4_b1_128k": (1, 8, 32, 131072, 2026),
}


@pytest.mark.parametrize("cfg", list(CONFIGS))
def test_full_size_sampled_units_every_chunk(cfg):
    B, Hkv, Hq, n, seed = CONFIGS[cfg]
    g = orc.rng(seed)
    k, v, q = _bf16((B, Hkv, n, D), g), _bf16((B, Hkv, n, D), g), _bf16((B, Hq, D), g)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    seeds = list(range(Hkv))
    cache.prefill(k.cuda(), v.cuda(), adapters=AdapterBank.initialize(Hkv, seeds=seeds))
    assert int(cache.n_chunks[0]) == (n - 128) // 128
    _check_units(cache, k, v, q, _sample_units(B, Hkv, 8, seed), seeds)


def test_config4_sequence_sharded_split_kv_on_one_gpu():
    """The split-KV path of distributed.SequenceShardedDecoder at config 4 (one 131k-token
    sequence), its ranks played by 4 shard caches on this GPU: each shard prefills its token
    range (keep_window=False except the tail owner), S / P are summed into the tail (the
    all-reduce), each shard emits one record per (b, q-head) over its own chunks
    (kvlc_decode_partial), the tail's correction row rides along, and kvlc_merge_records
    merges them.  Checked against the single-cache decode and, for two kv heads, against
    the oracle at T4."""
    from paper_2510_05373_b200.batched import merge_records
    from paper_2510_05373_b200.distributed import plan_sequence_shards
    B, Hkv, Hq, n, world = 1, 8, 32, 131072, 4
    g = orc.rng(2029)
    k, v, q = _bf16((B, Hkv, n, D), g), _bf16((B, Hkv, n, D), g), _bf16((B, Hq, D), g)
    seeds = list(range(Hkv))
    bank = AdapterBank.initialize(Hkv, seeds=seeds)
    kd, vd, qd = k.cuda(), v.cuda(), q.cuda()
    full = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    full.prefill(kd, vd, adapters=bank)
    ref_full = full.decode(qd, adapters=bank, out_dtype=torch.float32)
    shards = plan_sequence_shards(n, world)
    caches = []
    for sh in shards:
        c = BatchedKVCache(B, Hkv, Hq, max_tokens=sh.tok_hi - sh.tok_lo + 256)
        c.prefill(kd[:, :, sh.tok_lo:sh.tok_hi].contiguous(), vd[:, :, sh.tok_lo:sh.tok_hi].contiguous(),
                  adapters=bank, keep_window=sh.tail)
        assert int(c.n_chunks[0]) == sh.chunk_hi - sh.chunk_lo
        caches.append(c)
    tail = caches[-1]
    for c in caches[:-1]:  # the S / P all-reduce, into the tail owner
        tail.S += c.S
        tail.P += c.P
    recs, corr = [], None
    for sh, c in zip(shards, caches):
        rec, cr = c.decode_partial(qd, 0, int(c.n_chunks[0]), sh.tail, adapters=bank)
        recs.append(rec)
        if sh.tail:
            corr = cr
    merged = merge_records(torch.stack(recs), corr, out_dtype=torch.float32)
    e = (merged - ref_full).abs().max().item() / ref_full.abs().max().item()
    assert e <= 2e-4, e
    out = merged.cpu().numpy()
    qn = q.float().numpy().astype(np.float64)
    units = [(0, 0), (0, Hkv - 1)]
    NG = Hq // Hkv
    for (b, h), oc in zip(units, _oracle_caches(k, v, units, seeds)):
        ad = orc.init_adapter(D, 256, seed=seeds[h])
        ocm = orc.fp16_meta_copy(oc)
        for i in range(NG):
            ref = orc.decode_blocked(qn[b, h * NG + i], ocm, ad)
            err = np.abs(out[b, h * NG + i] - ref).max() / np.abs(ref).max()
            assert err <= OUT_TOL, (b, h, i, err)
