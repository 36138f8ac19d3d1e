"""Drop-in per-head streaming cache (quantkv.cache.KVCacheState, cache.py:49-194).

State lives in device memory (float64 residual window, packed u32 codes,
float64 scales/zeros, float64 S/P); `flush_group` is one call of the fused
`kvlc_ref_flush` kernel chain (channel-wise keys, FWHT-rotated token-wise
values, token-ordered S/P accumulation).  The attributes the reference
exposes (`key_chunks`, `value_rows`, `s_state`, ...) are materialised as host
arrays on access, so code written against the reference reads them
unchanged.

This per-head object is the reference-semantics path; the batched serving
cache is `paper_2510_05373_b200.batched.BatchedKVCache`.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import empty_dev, to_dev, to_host, zeros_dev
from .adapter import CorrectionAdapter
from .hadamard import hadamard_matrix
from .kvlc_format import VERSION, CacheFormatError, Header, join, parse_header, split
from .quantize import QuantConfig, QuantizedTensor, _lanes

__all__ = ["FootprintReport", "KVCacheState", "memory_footprint", "serialize_cache", "deserialize_cache",
           "write_cache", "read_cache", "CacheFormatError"]


@dataclass
class FootprintReport:
    """Serialized byte counts by component (header excluded), cache.py:35-46."""

    packed_codes: int
    scales_zeros: int
    residual: int
    correction_states: int

    @property
    def total(self) -> int:
        return self.packed_codes + self.scales_zeros + self.residual + self.correction_states


def _grow(t: torch.Tensor, need: int) -> torch.Tensor:
    """Capacity doubling along dim 0."""
    if t.shape[0] >= need:
        return t
    cap = max(need, 2 * t.shape[0], 4)
    out = torch.zeros((cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    out[: t.shape[0]] = t
    return out


class KVCacheState:
    """Per-head cache: packed history chunks, residual window, adapter states."""

    def __init__(self, head_dim: int, *, bits: int = 2, group_size: int = 128,
                 residual_window: int = 128, rotate_values: bool = True):
        if head_dim < 1:
            raise ValueError(f"head_dim must be >= 1, got {head_dim}")
        if group_size < 1:
            raise ValueError(f"group_size must be >= 1, got {group_size}")
        if residual_window < 0:
            raise ValueError(f"residual_window must be >= 0, got {residual_window}")
        if rotate_values:
            hadamard_matrix(head_dim)  # fails early on non-power-of-two dims
        self.head_dim = head_dim
        self.group_size = group_size
        self.residual_window = residual_window
        self.config_k = QuantConfig(bits=bits, group_size=group_size, axis="channel")
        self.config_v = QuantConfig(bits=bits, group_size=group_size, axis="token",
                                    rotation="post" if rotate_values else "none")
        lanes = _lanes(bits)
        self._kw = -(-group_size // lanes)            # words per key-chunk column
        self._vw = -(-head_dim // lanes)              # words per value row
        self._vg = -(-head_dim // group_size)         # value groups per row
        self._n_chunks = 0
        self._res_len = 0
        self._dev = None                               # allocated lazily (needs the GPU)
        self.adapter_rank = 0
        self.tokens_total = 0

    # -- device storage ---------------------------------------------------

    def _storage(self):
        if self._dev is None:
            d, g = self.head_dim, self.group_size
            cap = self.residual_window + g
            self._dev = {
                "res_k": zeros_dev((cap, d), "f64"),
                "res_v": zeros_dev((cap, d), "f64"),
                "kwords": zeros_dev((0, self._kw, d), "u32"),
                "kscales": zeros_dev((0, d), "f64"),
                "kzeros": zeros_dev((0, d), "f64"),
                "vwords": zeros_dev((0, self._vw), "u32"),
                "vscales": zeros_dev((0, self._vg), "f64"),
                "vzeros": zeros_dev((0, self._vg), "f64"),
                "s": None,
                "p": None,
            }
        return self._dev

    # -- views ------------------------------------------------------------

    @property
    def values_rotated(self) -> bool:
        return self.config_v.rotation == "post"

    @property
    def quantized_tokens(self) -> int:
        return self.group_size * self._n_chunks

    @property
    def residual_len(self) -> int:
        return self._res_len

    @property
    def key_chunks(self) -> list:
        if self._n_chunks == 0:
            return []
        st = self._storage()
        n = self._n_chunks
        words = to_host(st["kwords"][:n], "u32")
        scales = to_host(st["kscales"][:n], "f64")
        zeros = to_host(st["kzeros"][:n], "f64")
        return [QuantizedTensor(np.ascontiguousarray(words[i]), scales[i:i + 1].copy(),
                                zeros[i:i + 1].copy(), self.group_size, self.head_dim, self.config_k)
                for i in range(n)]

    @property
    def value_rows(self):
        if self._n_chunks == 0:
            return None
        st = self._storage()
        nq = self.quantized_tokens
        return QuantizedTensor(to_host(st["vwords"][:nq], "u32"), to_host(st["vscales"][:nq], "f64"),
                               to_host(st["vzeros"][:nq], "f64"), nq, self.head_dim, self.config_v)

    @property
    def s_state(self):
        st = self._dev
        return None if st is None or st["s"] is None else to_host(st["s"], "f64")

    @property
    def p_state(self):
        st = self._dev
        return None if st is None or st["p"] is None else to_host(st["p"], "f64")

    def residual_keys(self) -> np.ndarray:
        if self._res_len == 0:
            return np.zeros((0, self.head_dim))
        return to_host(self._storage()["res_k"][: self._res_len], "f64")

    def residual_values(self) -> np.ndarray:
        if self._res_len == 0:
            return np.zeros((0, self.head_dim))
        return to_host(self._storage()["res_v"][: self._res_len], "f64")

    def dequantized_keys(self, lo: int, hi: int) -> np.ndarray:
        """Dequantized key rows [lo, hi) of the quantized history (cache.py:97-105)."""
        self._check_range(lo, hi)
        g = self.group_size
        c0, c1 = lo // g, (hi - 1) // g + 1
        st = self._storage()
        d_out = empty_dev(((c1 - c0) * g, self.head_dim), "f64")
        for i, ci in enumerate(range(c0, c1)):
            _lib.call("kvlc_ref_dequantize", _lib.ptr(st["kwords"][ci]), _lib.ptr(st["kscales"][ci]),
                      _lib.ptr(st["kzeros"][ci]), g, self.head_dim, self.config_k.bits, g,
                      _lib.AXIS_CHANNEL, _lib.ptr(d_out[i * g:(i + 1) * g]), _lib.stream_handle())
        return to_host(d_out[lo - c0 * g: hi - c0 * g], "f64")

    def dequantized_values(self, lo: int, hi: int) -> np.ndarray:
        """Dequantized value rows [lo, hi) in the stored (possibly rotated) basis (cache.py:107-111)."""
        self._check_range(lo, hi)
        st = self._storage()
        d_out = empty_dev((hi - lo, self.head_dim), "f64")
        _lib.call("kvlc_ref_dequantize", _lib.ptr(st["vwords"][lo:hi]), _lib.ptr(st["vscales"][lo:hi]),
                  _lib.ptr(st["vzeros"][lo:hi]), hi - lo, self.head_dim, self.config_v.bits,
                  self.group_size, _lib.AXIS_TOKEN, _lib.ptr(d_out), _lib.stream_handle())
        return to_host(d_out, "f64")

    def _check_range(self, lo: int, hi: int):
        if not (0 <= lo < hi <= self.quantized_tokens):
            raise ValueError(f"token range [{lo}, {hi}) outside quantized "
                             f"history of {self.quantized_tokens}")

    # -- streaming --------------------------------------------------------

    def append(self, k_t, v_t, adapter: CorrectionAdapter | None = None):
        """Admit one token; flushes the oldest group when the window fills (cache.py:120-130)."""
        k_t = np.asarray(k_t, dtype=np.float64).reshape(-1)
        v_t = np.asarray(v_t, dtype=np.float64).reshape(-1)
        if k_t.shape != (self.head_dim,) or v_t.shape != (self.head_dim,):
            raise ValueError(f"token dims {k_t.shape}/{v_t.shape} != ({self.head_dim},)")
        st = self._storage()
        kv = to_dev(np.stack([k_t, v_t]))
        st["res_k"][self._res_len].copy_(kv[0])
        st["res_v"][self._res_len].copy_(kv[1])
        self._res_len += 1
        self.tokens_total += 1
        if self._res_len == self.residual_window + self.group_size:
            self.flush_group(adapter)

    def extend(self, k, v, adapter: CorrectionAdapter | None = None):
        """Append many tokens (same result as repeated `append`), one H2D copy per group."""
        k = np.asarray(k, dtype=np.float64)
        v = np.asarray(v, dtype=np.float64)
        if k.ndim != 2 or k.shape[1] != self.head_dim or v.shape != k.shape:
            raise ValueError(f"token dims {k.shape}/{v.shape} != (n, {self.head_dim})")
        st = self._storage()
        cap = self.residual_window + self.group_size
        i = 0
        while i < k.shape[0]:
            take = min(k.shape[0] - i, cap - self._res_len)
            st["res_k"][self._res_len:self._res_len + take].copy_(to_dev(k[i:i + take]))
            st["res_v"][self._res_len:self._res_len + take].copy_(to_dev(v[i:i + take]))
            self._res_len += take
            self.tokens_total += take
            i += take
            if self._res_len == cap:
                self.flush_group(adapter)

    def flush_group(self, adapter: CorrectionAdapter | None = None):
        """Quantize the oldest group_size residual tokens into the history (cache.py:132-158)."""
        g, d = self.group_size, self.head_dim
        if self._res_len < g:
            raise ValueError(f"need {g} residual tokens to flush, have {self._res_len}")
        st = self._storage()
        n, nq = self._n_chunks, self.quantized_tokens
        st["kwords"] = _grow(st["kwords"], n + 1)
        st["kscales"] = _grow(st["kscales"], n + 1)
        st["kzeros"] = _grow(st["kzeros"], n + 1)
        st["vwords"] = _grow(st["vwords"], nq + g)
        st["vscales"] = _grow(st["vscales"], nq + g)
        st["vzeros"] = _grow(st["vzeros"], nq + g)
        use = adapter is not None and adapter.enabled
        rank = adapter.rank if use else 0
        # The reference appends the chunk before validating the adapter
        # (cache.py:141-152), so a bad adapter still flushes; S/P stay untouched.
        error = None
        if use and adapter.head_dim != d:
            error = f"adapter dim {adapter.head_dim} != cache dim {d}"
        elif use and st["s"] is not None and self.adapter_rank != rank:
            error = f"adapter rank {rank} != cache state rank {self.adapter_rank}"
        with_states = use and error is None
        if with_states:
            self._ensure_states(rank)
            w1q, w2q, w1k, w2k = adapter.device_weights()
        scratch = empty_dev((_lib.load().kvlc_ref_flush_scratch(d, g, max(rank, 2)),), "u8")
        _lib.call("kvlc_ref_flush", _lib.ptr(st["res_k"]), _lib.ptr(st["res_v"]), d, g,
                  self.config_k.bits, int(self.values_rotated),
                  _lib.ptr(w1k) if with_states else None, _lib.ptr(w2k) if with_states else None,
                  rank, _lib.ptr(st["kwords"][n]), _lib.ptr(st["kscales"][n]),
                  _lib.ptr(st["kzeros"][n]), _lib.ptr(st["vwords"][nq]), _lib.ptr(st["vscales"][nq]),
                  _lib.ptr(st["vzeros"][nq]), _lib.ptr(st["s"]) if with_states else None,
                  _lib.ptr(st["p"]) if with_states else None, _lib.ptr(scratch),
                  _lib.stream_handle())
        rest = self._res_len - g
        if rest:
            st["res_k"][:rest] = st["res_k"][g:self._res_len].clone()
            st["res_v"][:rest] = st["res_v"][g:self._res_len].clone()
        self._res_len = rest
        self._n_chunks += 1
        if error is not None:
            raise ValueError(error)

    def _ensure_states(self, rank: int):
        st = self._storage()
        if st["s"] is None:
            self.adapter_rank = rank
            st["s"] = zeros_dev((self.head_dim, rank), "f64")
            st["p"] = zeros_dev((rank,), "f64")
        elif self.adapter_rank != rank:
            raise ValueError(f"adapter rank {rank} != cache state rank {self.adapter_rank}")


def memory_footprint(cache: KVCacheState) -> FootprintReport:
    """Exact serialized byte counts (cache.py:178-194): packed codes, 16-bit
    scales/zeros, 16-bit residual window, 16-bit correction states."""
    n, nq, d = cache._n_chunks, cache.quantized_tokens, cache.head_dim
    code_words = n * cache._kw * d + nq * cache._vw
    groups = n * d + nq * cache._vg
    states = 2 * (d * cache.adapter_rank + cache.adapter_rank) if cache.adapter_rank else 0
    return FootprintReport(packed_codes=4 * code_words, scales_zeros=2 * 2 * groups,
                           residual=2 * 2 * cache.residual_len * d, correction_states=states)


# -- serialization (cache.py:197-307) ------------------------------------------

def serialize_cache(cache: KVCacheState) -> bytes:
    """The reference's .kvlc bytes for one per-head cache (cache.py:209-230)."""
    n, d = cache._n_chunks, cache.head_dim
    h = Header(VERSION, d, cache.adapter_rank, cache.group_size, cache.residual_window,
               cache.config_k.bits, int(cache.values_rotated), cache.quantized_tokens, cache.residual_len)
    parts = {"res_k": cache.residual_keys(), "res_v": cache.residual_values()}
    if n:
        chunks = cache.key_chunks
        vr = cache.value_rows
        parts["kcodes"] = np.stack([c.codes for c in chunks])
        parts["kmeta"] = np.stack([np.stack([c.scales, c.zeros]) for c in chunks])
        parts.update(vcodes=vr.codes, vscales=vr.scales, vzeros=vr.zeros)
    else:
        for name, dt, shape in h.sections():
            parts.setdefault(name, np.zeros(shape))
    if cache.adapter_rank:
        parts["s"], parts["p"] = cache.s_state, cache.p_state
    return join(h, parts)


def deserialize_cache(data: bytes) -> KVCacheState:
    """Rebuild a per-head cache from .kvlc bytes (cache.py:252-307); the 16-bit
    fields come back as float64."""
    data = bytes(data)
    h = parse_header(data)
    cache = KVCacheState(h.head_dim, bits=h.bits, group_size=h.group, residual_window=h.window,
                         rotate_values=bool(h.rotated))
    sec = split(data, h)
    if h.n_res > h.window + h.group:
        raise CacheFormatError(f"residual length {h.n_res} exceeds window + group "
                               f"{h.window + h.group}")
    st = cache._storage()
    f64 = lambda a: np.asarray(a, np.float64)
    n = h.n_q // h.group
    if n:
        st["kwords"] = to_dev(np.ascontiguousarray(sec["kcodes"]).view(np.uint32).astype(np.uint32))
        st["kscales"] = to_dev(f64(sec["kmeta"][:, 0, 0]))
        st["kzeros"] = to_dev(f64(sec["kmeta"][:, 1, 0]))
        st["vwords"] = to_dev(np.ascontiguousarray(sec["vcodes"]).astype(np.uint32))
        st["vscales"] = to_dev(f64(sec["vscales"]))
        st["vzeros"] = to_dev(f64(sec["vzeros"]))
    if h.n_res:
        st["res_k"][: h.n_res] = to_dev(f64(sec["res_k"]))
        st["res_v"][: h.n_res] = to_dev(f64(sec["res_v"]))
    if h.rank:
        cache.adapter_rank = h.rank
        st["s"] = to_dev(f64(sec["s"]))
        st["p"] = to_dev(f64(sec["p"]))
    cache._n_chunks, cache._res_len = n, h.n_res
    cache.tokens_total = h.n_q + h.n_res
    return cache


def write_cache(cache: KVCacheState, path):
    """cache.py:310-312."""
    with open(path, "wb") as fh:
        fh.write(serialize_cache(cache))


def read_cache(path) -> KVCacheState:
    """cache.py:315-317."""
    with open(path, "rb") as fh:
        return deserialize_cache(fh.read())
