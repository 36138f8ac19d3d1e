"""Standalone block entry points (include/kvlinc.h "standalone blocks") vs the oracle.

kvlc_quantize_pack / kvlc_fwht_quantize_pack: packed words bit-exact (T1), fp16
scale / zero exactly float16(oracle float64) (T2), k_err / v_q equal to the
float64 oracle value rounded once to fp32.  kvlc_state_update: S, P within
1e-6 relative of the float64 loop (cache.py:155-158).  kvlc_flush_due: a deferred
flush leaves the cache byte-identical to the streaming append rule.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import kvlinc_oracle as orc  # noqa: E402
from paper_2510_05373_b200 import _lib  # noqa: E402
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
from kvlc_testutil import bf16_round  # noqa: E402

AXES = {"token": 0, "channel": 1}


def _bf16_dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).bfloat16().cuda()


def _meta_f16(a):
    return np.asarray(a, np.float64).astype(np.float16)


def _quantize_pack(x, bits, group, axis, ld=None, err=True):
    rows, cols = x.shape
    ld = ld or cols
    xp = np.zeros((rows, ld), np.float32)
    xp[:, :cols] = x
    xd = _bf16_dev(xp)
    L = orc.lanes_per_word(bits)
    if axis == "token":
        wshape, mshape = (rows, -(-cols // L)), (rows, -(-cols // group))
    else:
        wshape, mshape = (-(-rows // L), cols), (-(-rows // group), cols)
    words = torch.full(wshape, -1, dtype=torch.int32, device="cuda")  # garbage: kernel must own every word
    sc = torch.empty(mshape, dtype=torch.float16, device="cuda")
    ze = torch.empty(mshape, dtype=torch.float16, device="cuda")
    e = torch.empty((rows, cols), dtype=torch.float32, device="cuda") if err else None
    if group % L:
        words.zero_()
    _lib.call("kvlc_quantize_pack", xd.data_ptr(), rows, cols, ld, AXES[axis], bits, group, words.data_ptr(),
              sc.data_ptr(), ze.data_ptr(), _lib.ptr(e), _lib.stream_handle())
    torch.cuda.synchronize()
    return (words.cpu().numpy().view(np.uint32), sc.cpu().numpy(), ze.cpu().numpy(),
            None if e is None else e.cpu().numpy())


@pytest.mark.parametrize("axis", ["token", "channel"])
@pytest.mark.parametrize("bits,group,shape", [(2, 128, (128, 128)), (2, 128, (130, 77)), (3, 20, (37, 45)),
                                              (4, 32, (64, 96)), (8, 7, (19, 33)), (2, 20, (41, 50))])
def test_quantize_pack_matches_oracle(axis, bits, group, shape):
    g = orc.rng(bits * 100 + group)
    x = bf16_round(g.standard_normal(shape).astype(np.float32) * 3.0)
    x[0, : min(5, shape[1])] = x[0, 0]  # ties / repeated values
    words, sc, ze, err = _quantize_pack(x, bits, group, axis, ld=shape[1] + 3)
    ref = orc.quantize_matrix(x, bits, group, axis)
    assert np.array_equal(words, ref.words)
    assert np.array_equal(sc, _meta_f16(ref.scales)) and np.array_equal(ze, _meta_f16(ref.zeros))
    want = (x - orc.dequantize_matrix(ref)).astype(np.float32)
    assert np.array_equal(err, want)


def test_quantize_pack_key_chunk_and_degenerate_groups():
    """A serving key chunk (128 tokens x 128 channels, channel axis) with constant
    channels (scale 0 -> codes 0, quantize.py:205-207) and an exact grid."""
    g = orc.rng(5)
    x = bf16_round(g.standard_normal((128, 128)).astype(np.float32))
    x[:, 3] = 1.25
    x[:, 7] = np.tile([0.0, 1.0, 2.0, 3.0], 32)
    words, sc, ze, err = _quantize_pack(x, 2, 128, "channel")
    ref = orc.quantize_matrix(x, 2, 128, "channel")
    assert np.array_equal(words, ref.words)
    assert sc[0, 3] == 0 and np.all((words[:, 3]) == 0) and np.all(err[:, 3] == 0)
    assert np.all(err[:, 7] == 0)


def test_quantize_pack_rejects_like_reference():
    x = torch.zeros((4, 4), dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(16, dtype=torch.int32, device="cuda")
    m = torch.zeros(16, dtype=torch.float16, device="cuda")
    args = lambda rows, cols, bits, group: (x.data_ptr(), rows, cols, cols, 0, bits, group, w.data_ptr(),
                                            m.data_ptr(), m.data_ptr(), None, None)
    with pytest.raises(ValueError, match="passthrough"):
        _lib.call("kvlc_quantize_pack", *args(4, 4, 16, 4))
    with pytest.raises(ValueError, match="bits"):
        _lib.call("kvlc_quantize_pack", *args(4, 4, 5, 4))
    with pytest.raises(ValueError, match="non-empty"):
        _lib.call("kvlc_quantize_pack", *args(0, 4, 2, 4))


@pytest.mark.parametrize("bits,group,dim,rows", [(2, 128, 128, 128), (2, 128, 128, 77), (4, 32, 64, 50),
                                                 (3, 20, 32, 9)])
def test_fwht_quantize_pack_matches_oracle(bits, group, dim, rows):
    g = orc.rng(dim + rows)
    v = bf16_round(g.standard_normal((rows, dim)).astype(np.float32))
    v[1] = 0.5  # constant row -> (c sqrt(d), 0, ...) after rotation (test_hadamard.py:77-84)
    lib = _lib.load()
    ws = torch.empty(lib.kvlc_fwht_quantize_workspace(rows, dim), dtype=torch.uint8, device="cuda")
    L = orc.lanes_per_word(bits)
    words = torch.zeros((rows, -(-dim // L)), dtype=torch.int32, device="cuda")
    sc = torch.empty((rows, -(-dim // group)), dtype=torch.float16, device="cuda")
    ze = torch.empty_like(sc)
    vq = torch.empty((rows, dim), dtype=torch.float32, device="cuda")
    xd = _bf16_dev(v)
    _lib.call("kvlc_fwht_quantize_pack", xd.data_ptr(), rows, dim, dim, bits, group, words.data_ptr(),
              sc.data_ptr(), ze.data_ptr(), vq.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle())
    torch.cuda.synchronize()
    rot = orc.rotate_post(v)
    ref = orc.quantize_matrix(rot, bits, group, "token")
    assert np.array_equal(words.cpu().numpy().view(np.uint32), ref.words)
    assert np.array_equal(sc.cpu().numpy(), _meta_f16(ref.scales))
    assert np.array_equal(ze.cpu().numpy(), _meta_f16(ref.zeros))
    assert np.array_equal(vq.cpu().numpy(), orc.dequantize_matrix(ref).astype(np.float32))


@pytest.mark.parametrize("n,d,rank", [(128, 128, 256), (37, 64, 32)])
def test_state_update_matches_fp64_loop(n, d, rank):
    g = orc.rng(n)
    ad = orc.init_adapter(d, rank, seed=3)
    k_err = (g.standard_normal((n, d)) * 0.2).astype(np.float32)
    vq = g.standard_normal((n, d)).astype(np.float32)
    w1 = ad.w1_k.astype(np.float32)
    w2 = ad.w2_k.astype(np.float32)
    S0 = g.standard_normal((d, rank)).astype(np.float32)
    P0 = g.random(rank).astype(np.float32)
    lib = _lib.load()
    ws = torch.empty(lib.kvlc_state_update_workspace(n, rank), dtype=torch.uint8, device="cuda")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    S, P = t(S0), t(P0)
    dk, dv, dw1, dw2 = t(k_err), t(vq), t(w1), t(w2)  # keep the device copies alive across the call
    _lib.call("kvlc_state_update", dk.data_ptr(), dv.data_ptr(), n, d, rank, dw1.data_ptr(), dw2.data_ptr(),
              S.data_ptr(), P.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle())
    torch.cuda.synchronize()
    phi = orc.feature_map(k_err.astype(np.float64), w1.astype(np.float64), w2.astype(np.float64))
    S_ref, P_ref = S0.astype(np.float64), P0.astype(np.float64)
    for i in range(n):  # cache.py:155-158
        S_ref = S_ref + np.outer(vq[i].astype(np.float64), phi[i])
        P_ref = P_ref + phi[i]
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(S.cpu().numpy(), S_ref) < 1e-6 and rel(P.cpu().numpy(), P_ref) < 1e-6


def _flush_inputs(B, Hkv, n, seed):
    g = orc.rng(seed)
    k = bf16_round(g.standard_normal((n, B, Hkv, 128)).astype(np.float32))
    v = bf16_round(g.standard_normal((n, B, Hkv, 128)).astype(np.float32))
    return k, v


@pytest.mark.parametrize("use_adapter", [True, False])
def test_flush_due_equals_streaming_append(use_adapter):
    """Deferred appends + flush_due == the streaming rule (flush at R + G)."""
    B, Hkv, Hq, n = 3, 2, 8, 300
    k, v = _flush_inputs(B, Hkv, n, 9)
    bank = AdapterBank.initialize(Hkv) if use_adapter else None
    active = lambda i: np.array([True, i < 250, i % 2 == 0])
    a = BatchedKVCache(B, Hkv, Hq, 640)
    b = BatchedKVCache(B, Hkv, Hq, 640)
    flushed = np.zeros(B, np.int64)
    for i in range(n):
        kt, vt = _bf16_dev(k[i]), _bf16_dev(v[i])
        a.append(kt, vt, adapters=bank, active=active(i))
        b.append(kt, vt, adapters=bank, active=active(i), defer_flush=True)
        if np.any(b.res_len >= 256) or i % 7 == 6 or i == n - 1:  # batched, late flushes
            flushed += b.flush_due(adapters=bank)
    torch.cuda.synchronize()
    assert np.array_equal(a.n_chunks, b.n_chunks) and np.array_equal(a.res_len, b.res_len)
    assert flushed.tolist() == a.n_chunks.tolist() and a.n_chunks.tolist() == [1, 0, 0]
    for bb in range(B):
        for h in range(Hkv):
            for c in range(int(a.n_chunks[bb])):
                ea, eb = a.export_chunk(bb, h, c), b.export_chunk(bb, h, c)
                for key in ea:
                    assert np.array_equal(ea[key], eb[key]), key
            ka, va = a.residual(bb, h)
            kb, vb = b.residual(bb, h)
            assert np.array_equal(ka, kb) and np.array_equal(va, vb)
    assert torch.equal(a.S, b.S) and torch.equal(a.P, b.P)
    with pytest.raises(ValueError, match="flush_due"):
        for i in range(200):
            b.append(_bf16_dev(k[0]), _bf16_dev(v[0]), active=[True, False, False], defer_flush=True)
