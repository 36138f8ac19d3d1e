"""Batched serving path (fused flush + split-KV GQA decode) vs the CPU oracle.

Numerics contract:
  T1 packed code words, chunk / residual counters: bit-exact
  T2 fp16 scale / zero: exactly float16(reference float64 value)
  T3 S, P: relative Frobenius <= 1e-5 against the float64 reference states
  T4 decode output vs decode_step_blocked on the fp16-metadata oracle cache:
     max-abs <= 1e-3 * max|ref|
  T5 correction isolation: (out_adapter - out_plain) within 5% relative
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache, merge_records  # noqa: E402
from kvlc_testutil import bf16_round  # noqa: E402

D = 128
F32 = torch.float32


def make_inputs(B, Hkv, Hq, n, seed=0):
    g = orc.rng(seed)
    k = bf16_round(g.standard_normal((B, Hkv, n, D)).astype(np.float32))
    v = bf16_round(g.standard_normal((B, Hkv, n, D)).astype(np.float32))
    q = bf16_round(g.standard_normal((B, Hq, D)).astype(np.float32))
    return k, v, q


def tdev(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().to(torch.bfloat16)


def oracle_caches(k, v, lens, adapters):
    B, Hkv = k.shape[:2]
    return [[orc.build_cache(k[b, h, :lens[b]], v[b, h, :lens[b]],
                             adapters[h] if adapters else None) for h in range(Hkv)] for b in range(B)]


def check_cache_exact(cache, ocs, lens):
    B, Hkv = len(ocs), len(ocs[0])
    for b in range(B):
        oc0 = ocs[b][0]
        assert cache.n_chunks[b] == len(oc0.key_chunks)
        assert cache.res_len[b] == oc0.residual_len
        for h in range(Hkv):
            oc = ocs[b][h]
            for ci, ch in enumerate(oc.key_chunks):
                ex = cache.export_chunk(b, h, ci)
                assert np.array_equal(ex["kwords"], ch.words), (b, h, ci)
                assert np.array_equal(ex["kscale"], ch.scales[0].astype(np.float16)), (b, h, ci)
                assert np.array_equal(ex["kzero"], ch.zeros[0].astype(np.float16)), (b, h, ci)
                sl = slice(ci * 128, (ci + 1) * 128)
                assert np.array_equal(ex["vwords"], oc.value_words[sl]), (b, h, ci)
                assert np.array_equal(ex["vscale"], oc.value_scales[sl, 0].astype(np.float16)), (b, h, ci)
                assert np.array_equal(ex["vzero"], oc.value_zeros[sl, 0].astype(np.float16)), (b, h, ci)
            rk, rv = cache.residual(b, h)
            assert np.array_equal(rk, oc.residual_keys().astype(np.float32))
            assert np.array_equal(rv, oc.residual_values().astype(np.float32))


def check_states(cache, ocs):
    for b in range(len(ocs)):
        for h in range(len(ocs[0])):
            oc = ocs[b][h]
            u = b * cache.Hkv + h
            S = cache.S[u].double().cpu().numpy()
            P = cache.P[u].double().cpu().numpy()
            if oc.s_state is None:
                assert not S.any() and not P.any()
                continue
            assert np.linalg.norm(S - oc.s_state) <= 1e-5 * np.linalg.norm(oc.s_state), (b, h)
            assert np.linalg.norm(P - oc.p_state) <= 1e-5 * np.linalg.norm(oc.p_state), (b, h)


def oracle_decode(q, ocs, adapters, literal=False):
    B, Hq, _ = q.shape
    g = Hq // len(ocs[0])
    out = np.zeros((B, Hq, D))
    for b in range(B):
        for h in range(Hq):
            oc = orc.fp16_meta_copy(ocs[b][h // g])
            out[b, h] = orc.decode_blocked(q[b, h], oc, adapters[h // g] if adapters else None,
                                           literal=literal)
    return out


@pytest.mark.parametrize("Hkv,Hq,lens", [(2, 8, [900, 511]), (1, 7, [640]), (2, 2, [300, 1000]),
                                         (1, 8, [385]), (2, 4, [700, 257]), (1, 3, [520, 129, 1]),
                                         (2, 10, [600]), (1, 6, [1100, 384])])
def test_prefill_and_decode_vs_oracle(Hkv, Hq, lens):
    B = len(lens)
    n = max(lens)
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=Hq * 10 + B)
    oads = [orc.init_adapter(D, 256, seed=h) for h in range(Hkv)]
    bank = AdapterBank.initialize(Hkv)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    cache.prefill(tdev(k), tdev(v), lens=lens, adapters=bank)
    ocs = oracle_caches(k, v, lens, oads)
    check_cache_exact(cache, ocs, lens)
    check_states(cache, ocs)
    for literal in (False, True):
        out = cache.decode(tdev(q), adapters=bank, literal=literal, out_dtype=F32).cpu().numpy()
        ref = oracle_decode(q, ocs, oads, literal=literal)
        err = np.abs(out - ref).max()
        assert err <= 1e-3 * np.abs(ref).max(), (literal, err, np.abs(ref).max())
    plain = cache.decode(tdev(q), out_dtype=F32).cpu().numpy()
    ref_plain = oracle_decode(q, ocs, None)
    assert np.abs(plain - ref_plain).max() <= 1e-3 * np.abs(ref_plain).max()
    ref_ad = oracle_decode(q, ocs, oads)
    out_ad = cache.decode(tdev(q), adapters=bank, out_dtype=F32).cpu().numpy()
    delta_ref, delta = ref_ad - ref_plain, out_ad - plain
    if np.abs(delta_ref).max() > 0:
        assert np.abs(delta - delta_ref).max() <= 0.05 * np.abs(delta_ref).max() + 2e-3 * np.abs(ref_ad).max()


def test_append_stream_crosses_flushes():
    B, Hkv, Hq = 2, 2, 8
    lens0 = [250, 100]
    steps = 300
    n = max(lens0) + steps
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=7)
    oads = [orc.init_adapter(D, 256, seed=h) for h in range(Hkv)]
    bank = AdapterBank.initialize(Hkv)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    cache.prefill(tdev(k[:, :, :max(lens0)]), tdev(v[:, :, :max(lens0)]), lens=lens0, adapters=bank)
    pos = list(lens0)
    for s in range(steps):
        kt = np.stack([k[b, :, pos[b]] for b in range(B)])
        vt = np.stack([v[b, :, pos[b]] for b in range(B)])
        cache.append(tdev(kt), tdev(vt), adapters=bank)
        pos = [p + 1 for p in pos]
    lens = pos
    ocs = oracle_caches(k, v, lens, oads)
    check_cache_exact(cache, ocs, lens)
    check_states(cache, ocs)
    out = cache.decode(tdev(q), adapters=bank, out_dtype=F32).cpu().numpy()
    ref = oracle_decode(q, ocs, oads)
    assert np.abs(out - ref).max() <= 1e-3 * np.abs(ref).max()


def test_decode_right_after_flushing_append():
    # decode is launched with programmatic dependent launch and streams codes before its
    # griddepcontrol.wait; after an append that flushes, the library launches it without
    # the overlap.  No host sync between the steps: every output is read
    # at the end and checked against the oracle state of its step.
    B, Hkv, Hq = 2, 2, 8
    lens0 = [254, 126]
    steps = 4
    n = max(lens0) + steps
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=31)
    oads = [orc.init_adapter(D, 256, seed=h) for h in range(Hkv)]
    bank = AdapterBank.initialize(Hkv)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    cache.prefill(tdev(k[:, :, :max(lens0)]), tdev(v[:, :, :max(lens0)]), lens=lens0, adapters=bank)
    pos, outs, lens_at = list(lens0), [], []
    qd = tdev(q)
    for s in range(steps):
        kt = np.stack([k[b, :, pos[b]] for b in range(B)])
        vt = np.stack([v[b, :, pos[b]] for b in range(B)])
        cache.append(tdev(kt), tdev(vt), adapters=bank)   # step 1 flushes sequence 0 (R + G)
        pos = [p + 1 for p in pos]
        outs.append(cache.decode(qd, adapters=bank, out_dtype=F32))
        lens_at.append(list(pos))
    for out, lens in zip(outs, lens_at):
        ref = oracle_decode(q, oracle_caches(k, v, lens, oads), oads)
        assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3 * np.abs(ref).max(), lens


def test_split_partials_merge_equals_full_decode():
    B, Hkv, Hq, n = 2, 2, 8, 1500
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=3)
    bank = AdapterBank.initialize(Hkv)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    cache.prefill(tdev(k), tdev(v), lens=[n, n - 333], adapters=bank)
    qd = tdev(q)
    full = cache.decode(qd, adapters=bank, out_dtype=F32)
    nch = int(cache.n_chunks.max())
    for parts in (2, 3, 4):
        bounds = np.linspace(0, nch, parts + 1).astype(int)
        recs, corr = [], None
        for i in range(parts):
            tail = i == parts - 1
            rec, c = cache.decode_partial(qd, int(bounds[i]), int(bounds[i + 1]), tail, adapters=bank)
            recs.append(rec)
            if tail:
                corr = c
        merged = merge_records(torch.stack(recs), corr, out_dtype=F32)
        # different split boundaries change the fp32 summation order and each split's
        # lazy-rescale reference point, relative to which p * s_v becomes an fp16 hi / lo
        # MMA operand: ~1e-4 of max|out|, inside T4's 1e-3 (the oracle checks above)
        e = (merged - full).abs().max().item() / full.abs().max().item()
        assert e <= 2e-4, f"parts={parts} rel diff {e:.3e}"
        for literal in (True,):
            m2 = merge_records(torch.stack(recs), corr, literal=literal, out_dtype=F32)
            f2 = cache.decode(qd, adapters=bank, literal=literal, out_dtype=F32)
            e = (m2 - f2).abs().max().item() / f2.abs().max().item()
            assert e <= 2e-4, f"literal parts={parts} rel diff {e:.3e}"


@pytest.mark.parametrize("cpc", [1, 2, 3])
def test_explicit_split_plans_match_default(cpc):
    # cpc 1: 81 records per unit (> 64: the combine is fused into the last CTA of each
    # unit); cpc 2 / 3: 42 / 29 records (the PDL-chained combine kernel)
    B, Hkv, Hq, n = 2, 2, 8, 80 * 128
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=21)
    bank = AdapterBank.initialize(Hkv)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    cache.prefill(tdev(k), tdev(v), lens=[n, n - 1000], adapters=bank)
    qd = tdev(q)
    for literal in (False, True):
        ref = cache.decode(qd, adapters=bank, literal=literal, out_dtype=F32)
        out = cache.decode(qd, adapters=bank, literal=literal, out_dtype=F32, chunks_per_split=cpc)
        e = (out - ref).abs().max().item() / ref.abs().max().item()
        assert e <= 2e-4, f"cpc={cpc} literal={literal} rel diff {e:.3e}"  # see the merge test above


def test_correction_dominated_extremes():
    # all-ones keys, q = +-300: exp terms underflow and out ~ H^T C_n / C_d
    B, Hkv, Hq, n = 1, 1, 4, 700
    g = orc.rng(15)
    k = np.ones((B, Hkv, n, D))
    v = bf16_round(g.standard_normal((B, Hkv, n, D)).astype(np.float32))
    oads = [orc.init_adapter(D, 256, seed=0)]
    bank = AdapterBank.initialize(1)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    cache.prefill(tdev(k), tdev(v), adapters=bank)
    ocs = oracle_caches(k, v, [n], oads)
    for sign in (300.0, -300.0):
        q = np.full((B, Hq, D), sign)
        out = cache.decode(tdev(q), adapters=bank, out_dtype=F32).cpu().numpy()
        assert np.all(np.isfinite(out))
        ref = oracle_decode(q, ocs, oads)
        assert np.abs(out - ref).max() <= 1e-2 * max(1e-6, np.abs(ref).max())


def test_short_and_empty_windows():
    B, Hkv, Hq = 3, 1, 4
    lens = [1, 128, 255]  # residual only, exactly the window, window + G - 1
    n = max(lens)
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=11)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=512)
    cache.prefill(tdev(k), tdev(v), lens=lens)
    assert list(cache.n_chunks) == [0, 0, 0]
    ocs = oracle_caches(k, v, lens, None)
    out = cache.decode(tdev(q), out_dtype=F32).cpu().numpy()
    ref = oracle_decode(q, ocs, None)
    assert np.abs(out - ref).max() <= 1e-3 * np.abs(ref).max()
    with pytest.raises(ValueError, match="empty cache"):
        BatchedKVCache(1, 1, 4, max_tokens=256).decode(tdev(q[:1]))


def test_value_tie_tokens_match_reference_codes():
    """n=4096 / seed 4100 holds a genuine (x-min)/scale = 0.5 +- 1ulp value tie
    (chunk 14, token 39, channel 17).  The serving flush re-evaluates such
    tokens in the reference's arithmetic order, so every code matches."""
    g = orc.rng(4100)
    n = 4096
    k = bf16_round(g.standard_normal((1, 1, n, D)).astype(np.float32))
    v = bf16_round(g.standard_normal((1, 1, n, D)).astype(np.float32))
    q = bf16_round(g.standard_normal((1, 4, D)).astype(np.float32))
    cache = BatchedKVCache(1, 1, 4, max_tokens=n + 256)
    cache.prefill(tdev(k), tdev(v))
    ocs = oracle_caches(k, v, [n], None)
    check_cache_exact(cache, ocs, [n])
    out = cache.decode(tdev(q), out_dtype=F32).cpu().numpy()
    ref = oracle_decode(q, ocs, None)
    assert np.abs(out - ref).max() <= 1e-3 * np.abs(ref).max()


def test_host_output_graph_matches_device_output():
    """capture_decode(q_host=, out_host=): H2D q inside the graph, the combine writes
    the result into pinned host memory; equal to the device-output decode."""
    B, Hkv, Hq, n = 2, 2, 8, 700
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=12)
    bank = AdapterBank.initialize(Hkv)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    cache.prefill(tdev(k), tdev(v), lens=[n, n - 200], adapters=bank)
    want = cache.decode(tdev(q), adapters=bank).cpu()
    q_host = torch.from_numpy(q.astype(np.float32)).bfloat16().pin_memory()
    out_host = torch.zeros((B, Hq, D), dtype=torch.bfloat16).pin_memory()
    qd = torch.empty((B, Hq, D), dtype=torch.bfloat16, device="cuda")
    g, out = cache.capture_decode(qd, adapters=bank, q_host=q_host, out_host=out_host)
    assert out.data_ptr() == out_host.data_ptr()
    out_host.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out_host, want)
    with pytest.raises(ValueError, match="pinned"):
        cache.decode(tdev(q), adapters=bank, out=torch.empty((B, Hq, D), dtype=torch.bfloat16))


def test_serving_step_graph_equals_eager_steps():
    """capture_serving_step: append + decode replayed from CUDA graphs == the eager calls,
    step by step, through two flush boundaries (the flushing step replays its own graph,
    captured ahead by prepare() in the second period)."""
    B, Hkv, Hq = 2, 2, 8
    g = orc.rng(21)
    n0 = 300
    k = tdev(bf16_round(g.standard_normal((B, Hkv, n0, D)).astype(np.float32)))
    bank = AdapterBank.initialize(Hkv)
    a = BatchedKVCache(B, Hkv, Hq, max_tokens=1024)
    b = BatchedKVCache(B, Hkv, Hq, max_tokens=1024)
    a.prefill(k, k, adapters=bank)
    b.prefill(k, k, adapters=bank)
    q = torch.empty((B, Hq, D), dtype=torch.bfloat16, device="cuda")
    kt = torch.empty((B, Hkv, D), dtype=torch.bfloat16, device="cuda")
    vt = torch.empty_like(kt)
    step, out = a.capture_serving_step(q, kt, vt, adapters=bank)
    assert a.steps_until_flush() == 255 - (n0 - 128)

    def fill():
        q.copy_(tdev(g.standard_normal((B, Hq, D))))
        kt.copy_(tdev(g.standard_normal((B, Hkv, D))))
        vt.copy_(tdev(g.standard_normal((B, Hkv, D))))

    for period in range(2):
        if period:
            step.prepare()
        for i in range(a.steps_until_flush() + 1):   # the last step of the period flushes
            fill()
            step.replay()
            b.append(kt, vt, adapters=bank)
            want = b.decode(q, adapters=bank)
            assert torch.equal(out, want), (period, i)
        assert np.array_equal(a.res_len, b.res_len) and np.array_equal(a.n_chunks, b.n_chunks)
        assert torch.equal(a.S, b.S) and torch.equal(a.kcodes, b.kcodes)
    assert list(a.n_chunks) == [3, 3]


def test_ring_flush_tensor_core_and_simt_paths_agree():
    """Decode-time flushes: the tensor-core path (kvlc_append with its workspace) and the SIMT
    kernel (no workspace) produce identical code words / metadata and S, P within T3; both
    match the oracle."""
    B, Hkv, Hq, n = 2, 2, 8, 520
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=17)
    oads = [orc.init_adapter(D, 256, seed=h) for h in range(Hkv)]
    bank = AdapterBank.initialize(Hkv)
    caches = []
    for tc in (True, False):
        cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
        cache._tc_flush = tc
        for i in range(n):
            cache.append(tdev(k[:, :, i]), tdev(v[:, :, i]), adapters=bank)
        caches.append(cache)
    ocs = oracle_caches(k, v, [n] * B, oads)
    for cache in caches:
        check_cache_exact(cache, ocs, [n] * B)
        check_states(cache, ocs)
    assert torch.equal(caches[0].kcodes, caches[1].kcodes) and torch.equal(caches[0].vcodes, caches[1].vcodes)
    assert torch.equal(caches[0].vscale, caches[1].vscale) and torch.equal(caches[0].kzero, caches[1].kzero)


def _rotr2(w):
    w = w.astype(np.uint64)
    return (((w >> 2) | (w << 30)) & 0xFFFFFFFF).astype(np.uint32)


def test_documented_code_word_layout():
    """include/kvlinc.h documents the fragment-native kcodes / vcodes word layout; decode the
    raw device words with that formula and compare with kvlc_export_chunk (reference layout)."""
    B, Hkv, Hq, n = 1, 2, 8, 640
    k, v, _ = make_inputs(B, Hkv, Hq, n, seed=31)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 128)
    cache.prefill(tdev(k), tdev(v), adapters=AdapterBank.initialize(Hkv))
    nc = int(cache.n_chunks[0])
    assert nc >= 2
    koff, voff = [0, 8, 1, 9], [0, 1, 4, 5]
    for u in range(Hkv):
        for ci in range(nc):
            kw = _rotr2(cache.kcodes[u, ci].cpu().numpy().view(np.uint32).reshape(-1))
            vw = _rotr2(cache.vcodes[u, ci].cpu().numpy().view(np.uint32).reshape(-1))
            kc = np.zeros((128, 128), np.uint8)  # [token][channel]
            vc = np.zeros((128, 128), np.uint8)
            for wi in range(1024):
                w, lane, i = wi >> 8, (wi >> 3) & 31, wi & 7
                g, t0 = lane >> 2, lane & 3
                for q in range(4):
                    for j in range(4):
                        code_k = (kw[wi] >> (8 * q + 2 * j)) & 3
                        code_v = (vw[wi] >> (8 * q + 2 * j)) & 3
                        kc[32 * w + 4 * g + j, 16 * i + 2 * t0 + koff[q]] = code_k
                        vc[32 * w + 8 * t0 + 2 * (i >> 2) + voff[q], 32 * (i & 3) + 8 * j + g] = code_v
            ex = cache.export_chunk(0, u, ci)
            # reference layouts: key words (8, 128) tokens 16w.. of channel c; value rows (128, 8)
            want_k = np.zeros((8, 128), np.uint32)
            want_v = np.zeros((128, 8), np.uint32)
            for w in range(8):
                for l in range(16):
                    want_k[w] |= kc[16 * w + l].astype(np.uint32) << (2 * l)
            for jw in range(8):
                for l in range(16):
                    want_v[:, jw] |= vc[:, 16 * jw + l].astype(np.uint32) << (2 * l)
            assert np.array_equal(ex["kwords"], want_k), (u, ci)
            assert np.array_equal(ex["vwords"], want_v), (u, ci)


def test_decode_right_after_prefill_from_another_thread():
    """prefill writes codes and chunk counts that the decode reads before its
    griddepcontrol.wait.  The write mark lives with the cache (not the host thread or the
    stream), so a decode issued by another thread right after a prefill, with no host
    sync, still waits for it.  Two caches back to back in the same stream: prefill A,
    prefill B, decode A, decode B (each decode follows a writer of a different cache)."""
    import threading
    B, Hkv, Hq, n = 2, 2, 8, 700
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=41)
    oads = [orc.init_adapter(D, 256, seed=h) for h in range(Hkv)]
    bank = AdapterBank.initialize(Hkv)
    caches = [BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256) for _ in range(2)]
    kd, vd, qd = tdev(k), tdev(v), tdev(q)
    torch.cuda.synchronize()

    def writer():
        for c in caches:
            c.prefill(kd, vd, adapters=bank)

    th = threading.Thread(target=writer)
    th.start()
    th.join()  # host order only: the GPU work is still queued, nothing synchronised
    outs = [c.decode(qd, adapters=bank, out_dtype=F32) for c in caches]
    ref = oracle_decode(q, oracle_caches(k, v, [n] * B, oads), oads)
    for out in outs:
        assert np.abs(out.cpu().numpy() - ref).max() <= 1e-3 * np.abs(ref).max()


def test_captured_decode_refuses_a_changed_cache():
    """a capture_decode graph fixes the split plan and the workspace pointer;
    after a flush changes the chunk counts its replay raises instead of skipping chunks."""
    B, Hkv, Hq = 1, 1, 4
    k, v, q = make_inputs(B, Hkv, Hq, 255, seed=51)
    bank = AdapterBank.initialize(Hkv)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=1024)
    cache.prefill(tdev(k), tdev(v), adapters=bank)
    g, _ = cache.capture_decode(tdev(q), adapters=bank)
    g.replay()
    cache.append(tdev(k[:, :, :1]).reshape(B, Hkv, D), tdev(v[:, :, :1]).reshape(B, Hkv, D), adapters=bank)
    assert int(cache.n_chunks[0]) == 1   # 256 tokens: the append flushed a chunk
    with pytest.raises(ValueError, match="capture again"):
        g.replay()


@pytest.mark.parametrize("Hq,block", [(4, None), (8, None), (4, 256), (4, 384), (8, 512)])
def test_decode_blocks_match_reference_partials(Hq, block):
    """return_partials on the serving cache (kvlc_decode_blocks, block_tokens = G or a multiple):
    per-block (max, sum, y) against decode_step_blocked's DecodePartial on the oracle cache."""
    B, Hkv, n = 2, 2, 900
    lens = [900, 700]
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=61)
    oads = [orc.init_adapter(D, 256, seed=h) for h in range(Hkv)]
    bank = AdapterBank.initialize(Hkv)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    cache.prefill(tdev(k), tdev(v), lens=lens, adapters=bank)
    out, part = cache.decode_blocks(tdev(q), adapters=bank, block_tokens=block)
    full = cache.decode(tdev(q), adapters=bank, out_dtype=F32)
    assert (out - full).abs().max().item() <= 2e-4 * full.abs().max().item()
    ocs = oracle_caches(k, v, lens, oads)
    NG = Hq // Hkv
    for b in range(B):
        nbk = int(part["n_blocks"][b])
        for h in range(Hq):
            oc = orc.fp16_meta_copy(ocs[b][h // NG])
            _, (ry, rm, rl) = orc.decode_blocked(q[b, h].astype(np.float64), oc, oads[h // NG], block=block,
                                                 return_partials=True)
            assert len(rm) == nbk
            m = part["m"][b, h, :nbk].cpu().numpy()
            l = part["l"][b, h, :nbk].cpu().numpy()
            y = part["y"][b, h, :nbk].cpu().numpy()
            assert np.abs(m - rm).max() <= 1e-4 * max(1.0, np.abs(rm).max()), (b, h)
            assert np.abs(l - rl).max() <= 2e-4 * np.abs(rl).max(), (b, h)
            assert np.abs(y - ry).max() <= 1e-3 * np.abs(ry).max(), (b, h)
            assert not part["y"][b, h, nbk:].any()


def test_decode_blocks_rejects_partial_chunks():
    cache = BatchedKVCache(1, 1, 4, max_tokens=512)
    k, v, _ = make_inputs(1, 1, 4, 300, seed=3)
    cache.prefill(tdev(k), tdev(v))
    q = torch.zeros(1, 4, D, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="multiple of 128"):
        cache.decode_blocks(q, block_tokens=200)


def test_constant_value_rows_prefill_and_ring_flush():
    """Value rows whose channels are all equal (scale 0, codes 0): bit-exact metadata and the
    adapter state within T3 on the prefill path and on a decode-time ring flush (the state
    kernel stores such rows as s = 1, z' = z + 3/2 for its P / z'^T Phi MMA)."""
    B, Hkv, Hq, n = 1, 2, 8, 700
    k, v, q = make_inputs(B, Hkv, Hq, n, seed=29)
    # rows that are constant AFTER the value rotation: multiples of a unit vector (H e_0 is
    # flat) and zero rows
    v[:, :, 5:45, :] = 0.0
    v[:, :, 5:40, 0] = 0.5
    v[:, :, 300:330, :] = 0.0
    v[:, :, 300:330, 0] = -1.25
    oads = [orc.init_adapter(D, 256, seed=h) for h in range(Hkv)]
    bank = AdapterBank.initialize(Hkv)
    cache = BatchedKVCache(B, Hkv, Hq, max_tokens=n + 256)
    cache.prefill(tdev(k[:, :, :600]), tdev(v[:, :, :600]), adapters=bank)
    for i in range(600, n):
        cache.append(tdev(k[:, :, i]), tdev(v[:, :, i]), adapters=bank)
    ocs = oracle_caches(k, v, [n], oads)
    check_cache_exact(cache, ocs, [n])
    check_states(cache, ocs)
    out = cache.decode(tdev(q), adapters=bank, out_dtype=F32).cpu().numpy()
    ref = oracle_decode(q, ocs, oads)
    assert np.abs(out - ref).max() <= 1e-3 * np.abs(ref).max()
