"""Drop-in blocked decode step (quantkv.attention.decode_step_blocked,
attention.py:197-276) on the per-head device cache.

One call = the `kvlc_ref_decode` kernel chain: phi_q / correction states,
per-block float32 logits, max, exp, partial numerators, the ordered
shared-max block reduction with the e^{-M}-consistent (or literal)
correction (attention.py:158-194), the float32 H^T un-rotation and the
divide.  Batched GQA serving decode is `batched.BatchedKVCache.decode`.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import empty_dev, to_dev, to_host
from .adapter import CorrectionAdapter, _feature_map_dev
from .cache import KVCacheState
from .hadamard import hadamard_matrix, rotate
from .quantize import QuantConfig, quantize_tensor


@dataclass
class OpCounter:
    """Counts multiply-accumulates spent on correction terms (attention.py:30-37)."""

    macs: int = 0

    def add(self, n: int):
        self.macs += int(n)


@dataclass
class DecodePartial:
    """Per-block partial results of one blocked decode step (attention.py:41-47)."""

    y_partial: np.ndarray   # (blocks, d) float32, in the stored value basis
    block_max: np.ndarray   # (blocks,)
    block_sum: np.ndarray   # (blocks,)


def decode_step_blocked(q, cache: KVCacheState, adapter: CorrectionAdapter | None = None,
                        block_tokens: int | None = None, literal_correction: bool = False,
                        return_partials: bool = False):
    """One decode step over a streamed cache, block by block (attention.py:197-276)."""
    q = np.asarray(q, dtype=np.float64)
    d = cache.head_dim
    if q.shape != (d,):
        raise ValueError(f"query shape {q.shape} != head dim ({d},)")
    if cache.tokens_total == 0:
        raise ValueError("cannot decode against an empty cache")
    block = cache.group_size if block_tokens is None else block_tokens
    if block < 1:
        raise ValueError(f"block_tokens must be >= 1, got {block}")

    st = cache._storage()
    use_adapter = (adapter is not None and adapter.enabled and st["s"] is not None)
    rank = cache.adapter_rank if use_adapter else 0
    if use_adapter:
        w1q, w2q, _, _ = adapter.device_weights()
    nq, nr = cache.quantized_tokens, cache.residual_len
    nb = -(-nq // block) + (1 if nr else 0)
    lib = _lib.load()
    scratch = empty_dev((lib.kvlc_ref_decode_scratch(d, nq, nr, block, rank),), "u8")
    d_out = empty_dev((d,), "f64")
    py = empty_dev((max(nb, 1), d), "f32") if return_partials else None
    pm = empty_dev((max(nb, 1),), "f32") if return_partials else None
    pl = empty_dev((max(nb, 1),), "f32") if return_partials else None
    n_chunks = cache._n_chunks
    d_q = to_dev(q)
    _lib.call("kvlc_ref_decode", _lib.ptr(d_q), d, cache.group_size, cache.config_k.bits,
              int(cache.values_rotated), n_chunks,
              _lib.ptr(st["kwords"]), _lib.ptr(st["kscales"]), _lib.ptr(st["kzeros"]),
              _lib.ptr(st["vwords"]), _lib.ptr(st["vscales"]), _lib.ptr(st["vzeros"]),
              nr, _lib.ptr(st["res_k"]), _lib.ptr(st["res_v"]),
              _lib.ptr(w1q) if use_adapter else None, _lib.ptr(w2q) if use_adapter else None,
              _lib.ptr(st["s"]) if use_adapter else None, _lib.ptr(st["p"]) if use_adapter else None,
              rank, block, int(bool(literal_correction)), _lib.ptr(d_out),
              _lib.ptr(py), _lib.ptr(pm), _lib.ptr(pl), _lib.ptr(scratch), _lib.stream_handle())
    out = to_host(d_out, "f64")
    if return_partials:
        return out, DecodePartial(y_partial=to_host(py[:nb], "f32"), block_max=to_host(pm[:nb], "f32"),
                                  block_sum=to_host(pl[:nb], "f32"))
    return out


def quantize_roundtrip(x, cfg: QuantConfig) -> np.ndarray:
    """Rotate per config, quantize, dequantize, rotate back (attention.py:68-88): the
    matrix attention sees after storage, in the original basis; bits = 16 skips the
    quantization.  Every step runs on the device (kvlc_ref_rotate / _quantize /
    _dequantize); H is symmetric, so rotating back is the same rotation."""
    x = np.asarray(x, dtype=np.float64)
    if cfg.rotation == "pre":
        h = hadamard_matrix(x.shape[0])
        xr = rotate(x, h, "pre")
    elif cfg.rotation == "post":
        h = hadamard_matrix(x.shape[1])
        xr = rotate(x, h, "post")
    else:
        h, xr = None, x
    xq = xr if cfg.is_passthrough else quantize_tensor(xr, cfg).dequantize()
    if cfg.rotation == "pre":
        return rotate(xq, h, "pre")
    if cfg.rotation == "post":
        return rotate(xq, h, "post")
    return xq


# -- causal attention (prefill forms, attention.py:50-155) --------------------------

def _attention_dev(q, k, v, phq, phk, rank: int, shifted: bool, want_weights: bool):
    n, d = q.shape
    d_out = empty_dev((n, d), "f64")
    d_w = empty_dev((n, n), "f64") if want_weights else None
    d_q, d_k, d_v = to_dev(q), to_dev(k), to_dev(v)  # alive until the call has been enqueued and run
    _lib.call("kvlc_ref_attention", _lib.ptr(d_q), _lib.ptr(d_k), _lib.ptr(d_v), n, d,
              _lib.ptr(phq), _lib.ptr(phk), rank, int(shifted), _lib.ptr(d_w), _lib.ptr(d_out), _lib.stream_handle())
    return to_host(d_out, "f64"), (to_host(d_w, "f64") if want_weights else None)


def attention_reference(q_mat, k_mat, v_mat):
    """Full-precision causal attention (attention.py:50-57); returns (weights, outputs)."""
    q, k, v = (np.asarray(x, dtype=np.float64) for x in (q_mat, k_mat, v_mat))
    if q.shape != k.shape or k.shape != v.shape:
        raise ValueError(f"Q/K/V shapes differ: {q.shape} {k.shape} {v.shape}")
    out, w = _attention_dev(q, k, v, None, None, 0, shifted=True, want_weights=True)
    return w, out


def attention_with_config(q_mat, k_mat, v_mat, cfg_k: QuantConfig, cfg_v: QuantConfig):
    """Causal attention over quantize-roundtripped keys and values (attention.py:91-96)."""
    return attention_reference(q_mat, quantize_roundtrip(k_mat, cfg_k), quantize_roundtrip(v_mat, cfg_v))


def _corrected(q_mat, k_quant, k_err, v_quant, adapter):
    q, kq, vq = (np.asarray(x, dtype=np.float64) for x in (q_mat, k_quant, v_quant))
    n, d = q.shape
    use = adapter is not None and adapter.enabled
    phq = phk = None
    rank = 0
    if use:
        ke = np.asarray(k_err, dtype=np.float64)
        w1q, w2q, w1k, w2k = adapter.device_weights()
        h = adapter.rank // 2
        d_q, d_ke = to_dev(q), to_dev(ke)
        phq = _feature_map_dev(d_q, n, d, w1q, w2q, h)
        phk = _feature_map_dev(d_ke, n, d, w1k, w2k, h)
        rank = adapter.rank
    out, _ = _attention_dev(q, kq, vq, phq, phk, rank, shifted=False, want_weights=False)
    return out, use, n, d


def corrected_attention_quadratic(q_mat, k_quant, k_err, v_quant, adapter: CorrectionAdapter | None,
                                  counter: OpCounter | None = None):
    """Corrected causal attention, every f(q_n, k_err_i) explicit (attention.py:99-116):
    raw exponentials plus phi_q(q_n) . phi_k(k_err_i) over the causal prefix."""
    out, use, n, _ = _corrected(q_mat, k_quant, k_err, v_quant, adapter)
    if use and counter is not None:
        counter.add(n * (n + 1) // 2 * adapter.rank)
    return out


def corrected_attention_recurrent(q_mat, k_quant, k_err, v_quant, adapter: CorrectionAdapter | None,
                                  counter: OpCounter | None = None):
    """Same outputs as the quadratic form (attention.py:119-155); the reference's running
    (S, P) states are the prefix sums the kernel forms, and the counter charges the
    recurrent cost (phi_k, state update, phi_q, two contractions per token)."""
    out, use, n, d = _corrected(q_mat, k_quant, k_err, v_quant, adapter)
    if use and counter is not None:
        rank = adapter.rank
        counter.add(n * (4 * d * rank + 2 * rank))
    return out


# -- fast path: many heads, long prefixes (tensor cores) ------------------------------

def corrected_attention_batched(q, k_quant, k_err, v_quant, adapters=None):
    """corrected_attention_quadratic / _recurrent (attention.py:99-155) for many heads at
    once on the tensor cores (kvlc_corrected_attention): q, k_quant, k_err, v_quant are
    float32 [heads, n, 128] (torch tensors on the GPU, or arrays); adapters: one
    CorrectionAdapter (rank 256) per head, or None.  phi_q / phi_k come from the float64
    feature-map kernel.  Returns float32 [heads, n, 128] on the GPU.  Agrees with the float64
    reference forms to ~1e-5 of max|out| (fp16 hi / lo operands, fp32 accumulation)."""
    import torch
    dev = torch.device("cuda")
    f32 = lambda x: torch.as_tensor(x, dtype=torch.float32, device=dev).contiguous()
    q, kq, vq = f32(q), f32(k_quant), f32(v_quant)
    if q.dim() != 3 or q.shape != kq.shape or kq.shape != vq.shape or q.shape[2] != 128:
        raise ValueError(f"Q/K/V shapes differ or head dim != 128: {tuple(q.shape)} {tuple(kq.shape)} {tuple(vq.shape)}")
    heads, n, d = q.shape
    use = adapters is not None and any(a is not None and a.enabled for a in adapters)
    phq = phk = None
    rank = 0
    if use:
        if len(adapters) != heads or any(a is None or not a.enabled or a.rank != 256 for a in adapters):
            raise ValueError("one enabled rank-256 adapter per head")
        ke = f32(k_err)
        phq = torch.empty((heads, n, 256), dtype=torch.float32, device=dev)
        phk = torch.empty_like(phq)
        for h, ad in enumerate(adapters):
            w1q, w2q, w1k, w2k = ad.device_weights()
            xq = q[h].double().contiguous()
            xk = ke[h].double().contiguous()
            for src, w1, w2, dst in ((xq, w1q, w2q, phq), (xk, w1k, w2k, phk)):
                o = torch.empty((n, 256), dtype=torch.float64, device=dev)
                _lib.call("kvlc_ref_feature_map", src.data_ptr(), n, d, _lib.ptr(w1), _lib.ptr(w2), 128,
                          o.data_ptr(), _lib.stream_handle())
                dst[h].copy_(o)
        rank = 256
    out = torch.empty_like(q)
    nbytes = _lib.load().kvlc_corrected_attention_workspace(n, heads, rank)
    ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
    _lib.call("kvlc_corrected_attention", q.data_ptr(), kq.data_ptr(), vq.data_ptr(),
              phq.data_ptr() if use else None, phk.data_ptr() if use else None, n, heads, rank,
              out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle())
    return out
