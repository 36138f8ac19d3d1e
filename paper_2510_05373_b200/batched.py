"""Batched serving API: a [B, Hkv] 2-bit KVLinC cache on one B200.

Shapes are fixed at the production configuration the fast kernels
specialise on: head_dim d = 128, group G = 128, residual window R = 128,
adapter rank D = 256, 2-bit codes; GQA groups of 1..8 query heads per KV
head.  Activations (q, k, v, out) are bf16; scales / zeros are fp16 (the
.kvlc on-disk precision, cache.py:220-224); S / P are fp32.

    cache = BatchedKVCache(batch=16, kv_heads=8, q_heads=32, max_tokens=8192)
    bank = AdapterBank.initialize(kv_heads=8)          # one adapter per kv head
    cache.prefill(k, v, adapters=bank)                 # k, v: [B, Hkv, N, 128] bf16
    out = cache.decode(q, adapters=bank)               # q: [B, Hq, 128] bf16
    cache.append(k_t, v_t, adapters=bank)              # one token per sequence

Per (b, kv-head) the semantics are those of the reference's KVCacheState +
decode_step_blocked (cache.py:120-158, attention.py:197-276) with
query head h reading kv head h // (Hq // Hkv).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from . import kvlc_format as fmt
from ._lib import D, G, R, RANK, SLOTS, KvlcAdapter, KvlcCache, KvlcDecodeOpts
from .adapter import CorrectionAdapter

REC_FLOATS = 4 + 2 * D      # device-partial record: m_log2, l, 0, 0, y_rot[D], y_raw[D]
CORR_FLOATS = 1 + D         # correction record: C_d, C_n[D]


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class AdapterBank:
    """One CorrectionAdapter per kv head, fp32 device weights [Hkv][128][128]."""

    def __init__(self, adapters, enabled: bool = True, device=None):
        _lib.require_device()
        dev = device or torch.device("cuda", torch.cuda.current_device())
        for ad in adapters:
            if ad.head_dim != D or ad.rank != RANK:
                raise ValueError(f"serving adapters must be d={D}, rank={RANK}; got "
                                 f"d={ad.head_dim}, rank={ad.rank}")
        stack = lambda name: torch.from_numpy(np.stack([getattr(a, name) for a in adapters])
                                              .astype(np.float32)).to(dev).contiguous()
        self.adapters = list(adapters)
        self.w1q, self.w2q = stack("w1_q"), stack("w2_q")
        self.w1k, self.w2k = stack("w1_k"), stack("w2_k")
        self.enabled = enabled and all(a.enabled for a in adapters)

    @classmethod
    def initialize(cls, kv_heads: int, seeds=None, init_scale: float = 1.0, device=None):
        """Random-init adapters, seed = kv-head index by default."""
        seeds = list(range(kv_heads)) if seeds is None else list(seeds)
        return cls([CorrectionAdapter.initialize(D, RANK, seed=s, init_scale=init_scale)
                    for s in seeds], device=device)

    def struct(self) -> KvlcAdapter:
        return KvlcAdapter(self.w1q.data_ptr(), self.w2q.data_ptr(), self.w1k.data_ptr(),
                           self.w2k.data_ptr(), int(self.enabled))


def flush_count(lens, keep_window: bool = True) -> np.ndarray:
    """Chunks flushed after `lens` streaming appends: floor((len - R) / G) for
    len >= R (the flush fires when the window holds R + G tokens,
    cache.py:129), or floor(len / G) when no window is kept."""
    lens = np.asarray(lens, np.int64)
    if keep_window:
        return np.where(lens >= R, (lens - R) // G, 0)
    return lens // G


def _adapters_on(adapters) -> bool:
    return adapters is not None and bool(adapters.enabled)


def _adapter_struct(adapters):
    if adapters is None:
        return KvlcAdapter(None, None, None, None, 0)
    return adapters.struct()


class _GuardedGraph:
    """A captured decode step: the split plan and the decode workspace pointer
    are fixed at capture, so replay refuses to run once the cache's chunk counts or its
    decode workspace changed (a flush, or a later decode that grew the workspace)."""

    def __init__(self, graph, cache):
        self.graph, self.cache = graph, cache
        self.chunks = cache.n_chunks.copy()
        self.dws = cache._dws

    def replay(self):
        if not np.array_equal(self.chunks, self.cache.n_chunks) or self.cache._dws is not self.dws:
            raise ValueError("the cache changed since capture_decode (chunk counts or decode workspace): "
                             "capture again")
        self.graph.replay()


class BatchedKVCache:
    """Device-resident [B, Hkv] KVLinC cache (layout: include/kvlinc.h `kvlc_cache`)."""

    def __init__(self, batch: int, kv_heads: int, q_heads: int, max_tokens: int, device=None):
        _lib.require_device()
        if q_heads % kv_heads or q_heads // kv_heads > 8:
            raise ValueError(f"q_heads {q_heads} must be a multiple of kv_heads {kv_heads} "
                             "with at most 8 query heads per kv head")
        if batch > 1024:
            raise ValueError("batch must be <= 1024")
        self.B, self.Hkv, self.Hq = batch, kv_heads, q_heads
        self.group = q_heads // kv_heads
        self.max_tokens = max_tokens
        self.max_chunks = max(1, -(-max(0, max_tokens - R) // G))
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        U, C = batch * kv_heads, self.max_chunks
        z = lambda shape, dt: torch.zeros(shape, dtype=dt, device=dev)
        self.kcodes = z((U, C, 8, 128), torch.int32)
        self.vcodes = z((U, C, 8, 128), torch.int32)
        self.kscale = z((U, C, 128), torch.float16)
        self.kzero = z((U, C, 128), torch.float16)
        self.vscale = z((U, C, 128), torch.float16)
        self.vzero = z((U, C, 128), torch.float16)
        self.kres = z((U, SLOTS, D), torch.bfloat16)
        self.vres = z((U, D, SLOTS), torch.bfloat16)
        self.S = z((U, D, RANK), torch.float32)
        self.P = z((U, RANK), torch.float32)
        self.n_chunks_dev = z((batch,), torch.int32)
        self.res_start_dev = z((batch,), torch.int32)
        self.res_len_dev = z((batch,), torch.int32)
        # host mirror of the per-sequence counters (the host drives flushes)
        self.n_chunks = np.zeros(batch, np.int64)
        self.res_start = np.zeros(batch, np.int64)
        self.res_len = np.zeros(batch, np.int64)
        # adapter_rank of each sequence's states (cache.py:160-166): RANK after
        # its first flush with an enabled adapter, else 0 (no S / P in .kvlc)
        self.state_rank = np.zeros(batch, np.int64)
        self._ws = None
        self._struct = self._make_struct()

    # ------------------------------------------------------------------ plumbing
    def _make_struct(self) -> KvlcCache:
        p = lambda t: t.data_ptr()
        return KvlcCache(self.B, self.Hkv, self.Hq, self.max_chunks, p(self.kcodes), p(self.vcodes),
                         p(self.kscale), p(self.kzero), p(self.vscale), p(self.vzero), p(self.kres),
                         p(self.vres), p(self.S), p(self.P), p(self.n_chunks_dev),
                         p(self.res_start_dev), p(self.res_len_dev))

    def _flush_ws(self, flush, adapters):
        """(pointer, bytes) of the tensor-core flush workspace when an adapter flush is due
        (`_tc_flush = False` keeps the SIMT flush kernel: tests compare the two)."""
        if not np.any(flush) or not _adapters_on(adapters) or not getattr(self, "_tc_flush", True):
            return None, 0
        ws = self.workspace(_lib.load().kvlc_append_workspace(ctypes.byref(self._struct)))
        return _ptr(ws), ws.numel()

    def workspace(self, nbytes: int) -> torch.Tensor:
        """Scratch for prefill / append (contents are transient)."""
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=self.device)
        return self._ws

    def decode_ws(self, nbytes: int) -> torch.Tensor:
        """Decode workspace: zero-filled once; its head holds the per-unit arrival
        counters of the fused combine, which every decode launch leaves at zero."""
        if getattr(self, "_dws", None) is None or self._dws.numel() < nbytes:
            self._dws = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=self.device)
        return self._dws

    @property
    def tokens(self) -> np.ndarray:
        return self.n_chunks * G + self.res_len

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in
                   (self.kcodes, self.vcodes, self.kscale, self.kzero, self.vscale, self.vzero,
                    self.kres, self.vres, self.S, self.P))

    # ------------------------------------------------------------------ writers
    def prefill(self, k: torch.Tensor, v: torch.Tensor, lens=None, adapters: AdapterBank | None = None,
                keep_window: bool = True):
        """Load N tokens per sequence (== N streaming appends, cache.py:120-130).

        k, v: bf16 [B, Hkv, N, 128] (device or host).  lens: per-sequence
        token counts (default N).  keep_window=False flushes every whole
        chunk (a non-tail shard of a sequence-parallel cache, see
        `distributed`).  The cache must be empty."""
        if np.any(self.tokens):
            raise ValueError("prefill needs an empty cache")
        if k.shape != v.shape or k.dim() != 4 or k.shape[:2] != (self.B, self.Hkv) or k.shape[3] != D:
            raise ValueError(f"token dims {tuple(k.shape)}/{tuple(v.shape)} != ({self.B}, {self.Hkv}, n, {D})")
        n = k.shape[2]
        lens = np.full(self.B, n, np.int32) if lens is None else np.asarray(lens, np.int32)
        k = k.to(self.device, torch.bfloat16).contiguous()
        v = v.to(self.device, torch.bfloat16).contiguous()
        lib = _lib.load()
        ws = self.workspace(lib.kvlc_prefill_workspace(ctypes.byref(self._struct), n))
        ad = _adapter_struct(adapters)
        lens_c = (ctypes.c_int32 * self.B)(*lens.tolist())
        _lib.call("kvlc_prefill", ctypes.byref(self._struct), ctypes.byref(ad), _ptr(k), _ptr(v), n,
                  lens_c, int(bool(keep_window)), _ptr(ws), ws.numel(), _lib.stream_handle())
        nf = flush_count(lens, keep_window)
        if _adapters_on(adapters):
            self.state_rank[nf > 0] = RANK
        self.n_chunks[:] = nf
        self.res_start[:] = 0
        self.res_len[:] = lens - nf * G

    def append(self, k_t: torch.Tensor, v_t: torch.Tensor, adapters: AdapterBank | None = None,
               active=None, defer_flush: bool = False):
        """Append one token per (active) sequence: k_t, v_t bf16 [B, Hkv, 128].
        A sequence whose window reaches R + G flushes its oldest G tokens, unless
        `defer_flush` (the caller then runs `flush_due()` before that sequence's
        next append, e.g. to batch flushes off the decode step)."""
        if k_t.shape != (self.B, self.Hkv, D) or v_t.shape != k_t.shape:
            raise ValueError(f"token dims {tuple(k_t.shape)}/{tuple(v_t.shape)} != ({self.B}, {self.Hkv}, {D})")
        act = np.ones(self.B, bool) if active is None else np.asarray(active, bool)
        new_len = self.res_len + act
        if np.any(new_len > SLOTS):
            raise ValueError("residual window full: run flush_due() before appending")
        flush = act & (new_len == R + G) & (not defer_flush)
        if np.any(self.n_chunks + flush > self.max_chunks):
            raise ValueError(f"append exceeds capacity of {self.max_tokens} tokens")
        ad = _adapter_struct(adapters)
        a_c = (ctypes.c_int32 * self.B)(*act.astype(np.int32).tolist())
        f_c = (ctypes.c_int32 * self.B)(*flush.astype(np.int32).tolist())
        k_t = k_t.to(self.device, torch.bfloat16).contiguous()
        v_t = v_t.to(self.device, torch.bfloat16).contiguous()
        ws, nws = self._flush_ws(flush, adapters)
        _lib.call("kvlc_append", ctypes.byref(self._struct), ctypes.byref(ad), _ptr(k_t), _ptr(v_t),
                  a_c, f_c, ws, nws, _lib.stream_handle())
        if _adapters_on(adapters):
            self.state_rank[flush] = RANK
        self.res_len = new_len - flush * G
        self.res_start = np.where(flush, (self.res_start + G) % SLOTS, self.res_start)
        self.n_chunks = self.n_chunks + flush

    # ------------------------------------------------------------------ decode
    def _opts(self, literal=False, chunks_per_split=0, out_fp32=False, events=None) -> KvlcDecodeOpts:
        ev0, ev1 = (events[0].cuda_event, events[1].cuda_event) if events else (None, None)
        return KvlcDecodeOpts(int(chunks_per_split), int(bool(literal)), int(self.n_chunks.max()),
                              int(bool(out_fp32)), ev0, ev1)

    def decode_workspace_bytes(self, literal=False, chunks_per_split=0) -> int:
        o = self._opts(literal, chunks_per_split)
        return _lib.load().kvlc_decode_workspace(ctypes.byref(self._struct), ctypes.byref(o))

    def decode(self, q: torch.Tensor, adapters: AdapterBank | None = None, literal: bool = False,
               out: torch.Tensor | None = None, chunks_per_split: int = 0,
               out_dtype: torch.dtype = torch.bfloat16, events=None) -> torch.Tensor:
        """Fused GQA decode step: q bf16 [B, Hq, 128] -> out [B, Hq, 128] (bf16, or
        float32 with out_dtype=torch.float32).  events=(begin, end) torch.cuda.Event
        pair recorded around the split-KV kernel (measurement hook)."""
        if q.shape != (self.B, self.Hq, D):
            raise ValueError(f"query shape {tuple(q.shape)} != ({self.B}, {self.Hq}, {D})")
        if np.any(self.tokens == 0):
            raise ValueError("cannot decode against an empty cache")
        q = q.to(self.device, torch.bfloat16).contiguous()
        if out is None:
            out = torch.empty(q.shape, dtype=out_dtype, device=self.device)
        if out.dtype not in (torch.bfloat16, torch.float32) or out.shape != q.shape or not out.is_contiguous():
            raise ValueError("out must be a contiguous [B, Hq, 128] bf16 or float32 tensor")
        if out.device.type == "cpu" and not out.is_pinned():
            raise ValueError("a host `out` must be pinned (the kernel writes it through unified addressing)")
        o = self._opts(literal, chunks_per_split, out.dtype == torch.float32, events)
        nbytes = _lib.load().kvlc_decode_workspace(ctypes.byref(self._struct), ctypes.byref(o))
        ws = self.decode_ws(nbytes)
        ad = _adapter_struct(adapters)
        _lib.call("kvlc_decode", ctypes.byref(self._struct), ctypes.byref(ad), _ptr(q), _ptr(out),
                  ctypes.byref(o), _ptr(ws), ws.numel(), _lib.stream_handle())
        return out

    def decode_blocks(self, q: torch.Tensor, adapters: AdapterBank | None = None, literal: bool = False,
                      block_tokens: int | None = None):
        """decode_step_blocked(..., block_tokens, return_partials=True) for every (b, q-head)
        (attention.py:41-47, 197-276; kvlc_decode_blocks): returns (out float32 [B, Hq, 128],
        partials) with partials = dict(y [B, Hq, NB, 128] stored basis, m [B, Hq, NB] block max
        in natural logit units, l [B, Hq, NB] block sums, n_blocks [B]) -- the quantized blocks
        then the residual window as one block; rows past a sequence's n_blocks are zero.  The
        serving cache's blocks are whole chunks: block_tokens a multiple of G (default G); the
        per-head shim (attention.decode_step_blocked) takes any block size."""
        if q.shape != (self.B, self.Hq, D):
            raise ValueError(f"query shape {tuple(q.shape)} != ({self.B}, {self.Hq}, {D})")
        if np.any(self.tokens == 0):
            raise ValueError("cannot decode against an empty cache")
        block = G if block_tokens is None else int(block_tokens)
        if block < 1:
            raise ValueError(f"block_tokens must be >= 1, got {block}")
        if block % G:
            raise ValueError(f"the serving cache decodes whole chunks: block_tokens must be a multiple of {G}, "
                             f"got {block}")
        cpb = block // G
        q = q.to(self.device, torch.bfloat16).contiguous()
        out = torch.empty(q.shape, dtype=torch.float32, device=self.device)
        nb = -(-int(self.n_chunks.max()) // cpb) + 1
        blocks = torch.zeros((self.B, self.Hq, nb, 2 + D), dtype=torch.float32, device=self.device)
        o = self._opts(literal, cpb, True)
        nbytes = _lib.load().kvlc_decode_workspace(ctypes.byref(self._struct), ctypes.byref(o))
        ws = self.decode_ws(nbytes)
        ad = _adapter_struct(adapters)
        _lib.call("kvlc_decode_blocks", ctypes.byref(self._struct), ctypes.byref(ad), _ptr(q), _ptr(out),
                  _ptr(blocks), nb, ctypes.byref(o), _ptr(ws), ws.numel(), _lib.stream_handle())
        n_blocks = -(-self.n_chunks // cpb) + (self.res_len > 0)
        return out, {"m": blocks[..., 0], "l": blocks[..., 1], "y": blocks[..., 2:], "n_blocks": n_blocks}

    def capture_decode(self, q: torch.Tensor, adapters: AdapterBank | None = None, literal: bool = False,
                       out: torch.Tensor | None = None, chunks_per_split: int = 0,
                       q_host: torch.Tensor | None = None, out_host: torch.Tensor | None = None):
        """Capture one decode step on fixed q / out buffers into a CUDA graph (one
        graph launch per step).  With a pinned `q_host` the graph also holds the
        step's H2D copy of q (kvlc_stage_input, chained to the decode by programmatic
        dependent launch); with a pinned `out_host` the kernel's combine writes
        the result straight into host memory (unified addressing, no D2H copy node:
        a D2H copy after an H2D copy on one stream costs ~10 us of direction switch).
        Returns (graph, out); refill q (or q_host) in place and call graph.replay()."""
        if out_host is not None:
            out = out_host
        elif out is None:
            out = torch.empty(q.shape, dtype=torch.bfloat16, device=self.device)
        self.decode(q, adapters, literal, out, chunks_per_split)   # sizes the workspace
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        if q_host is not None and (q_host.dtype != torch.bfloat16 or q_host.shape != q.shape
                                   or not q_host.is_pinned() or not q_host.is_contiguous()):
            raise ValueError("q_host must be a pinned contiguous bf16 tensor shaped like q")
        with torch.cuda.graph(graph):
            if q_host is not None:   # copy kernel, programmatic-launch chained to the decode
                _lib.call("kvlc_stage_input", q_host.data_ptr(), q.data_ptr(), q.numel() * 2,
                          _lib.stream_handle())
            self.decode(q, adapters, literal, out, chunks_per_split)
        return _GuardedGraph(graph, self), out

    def steps_until_flush(self) -> int:
        """Appends every sequence can take before one of them reaches R + G (flushes)."""
        return int(np.min(R + G - 1 - self.res_len))

    def capture_serving_step(self, q: torch.Tensor, k_t: torch.Tensor, v_t: torch.Tensor,
                             adapters: AdapterBank | None = None, out: torch.Tensor | None = None):
        """Decode-loop steps as CUDA graph launches: append k_t, v_t (one token per
        sequence, cache.py:120-130) then the fused decode of q.  A step on which some
        sequences reach R + G replays a graph that also flushes them (kvlc_append with the
        tensor-core ring flush, cache.py:132-158).  The decode plan depends on the chunk
        counts, so graphs are keyed by (flush mask, chunk counts) and captured on first
        use; `.prepare()` captures the next flushing step's graph and the steady-state
        graph after it ahead of time.  Refill q / k_t / v_t in place and call `.replay()`;
        each replay advances the host mirrors (lengths, ring start, chunk counts)."""
        if k_t.shape != (self.B, self.Hkv, D) or v_t.shape != k_t.shape:
            raise ValueError(f"token dims {tuple(k_t.shape)}/{tuple(v_t.shape)} != ({self.B}, {self.Hkv}, {D})")
        if out is None:
            out = torch.empty(q.shape, dtype=torch.bfloat16, device=self.device)
        cache = self
        ad_on = _adapters_on(adapters)
        # workspaces sized once (largest plan up to capacity, the tensor-core flush) so the
        # pointers baked into captured graphs stay valid
        saved = cache.n_chunks
        need = 0
        for nc in range(int(saved.min()), cache.max_chunks + 1):
            cache.n_chunks = np.full_like(saved, nc)
            need = max(need, cache.decode_workspace_bytes())
        cache.n_chunks = saved
        dws = cache.decode_ws(need)
        fws = cache.workspace(_lib.load().kvlc_append_workspace(ctypes.byref(cache._struct))) if ad_on else None

        def due():
            return (cache.res_len + 1 == R + G).astype(np.int32)

        def capture(mask):
            m = (tuple(mask.tolist()), tuple(cache.n_chunks.tolist()))
            ad = _adapter_struct(adapters)
            a_c = (ctypes.c_int32 * cache.B)(*([1] * cache.B))
            f_c = (ctypes.c_int32 * cache.B)(*mask.tolist())
            tc = ad_on and np.any(mask) and getattr(cache, "_tc_flush", True)
            saved_n = cache.n_chunks
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(graph):
                    _lib.call("kvlc_append", ctypes.byref(cache._struct), ctypes.byref(ad), _ptr(k_t), _ptr(v_t),
                              a_c, f_c, _ptr(fws) if tc else None, fws.numel() if tc else 0,
                              _lib.stream_handle())
                    cache.n_chunks = saved_n + mask   # the decode's plan: counts after this step
                    cache.decode(q, adapters, out=out)
            finally:
                cache.n_chunks = saved_n
            if cache._dws is not dws:
                raise RuntimeError("decode workspace reallocated during capture")
            return m, graph

        class _Step:
            def __init__(self):
                self.graphs = {}

            def _graph(self, mask):
                key = (tuple(mask.tolist()), tuple(cache.n_chunks.tolist()))
                if key not in self.graphs:
                    if len(self.graphs) >= 4:
                        self.graphs.pop(next(iter(self.graphs)))
                    k2, g = capture(mask)
                    self.graphs[k2] = g
                return self.graphs[key]

            def replay(self):
                mask = due()
                self._graph(mask).replay()
                cache.res_len = cache.res_len + 1 - mask * G
                cache.res_start = np.where(mask > 0, (cache.res_start + G) % SLOTS, cache.res_start)
                cache.n_chunks = cache.n_chunks + mask
                if ad_on:
                    cache.state_rank[mask > 0] = RANK

            def prepare(self):
                """Capture (without running) the graphs of the next flushing step and of the
                steady state right after it."""
                saved = (cache.res_len, cache.res_start, cache.n_chunks)
                try:
                    steps = cache.steps_until_flush()
                    cache.res_len = cache.res_len + steps
                    mask = due()
                    self._graph(mask)
                    cache.res_len = cache.res_len + 1 - mask * G
                    cache.n_chunks = cache.n_chunks + mask
                    self._graph(due())
                finally:
                    cache.res_len, cache.res_start, cache.n_chunks = saved

        step = _Step()
        step._graph(due())
        return step, out

    def decode_partial(self, q: torch.Tensor, chunk_lo: int, chunk_hi: int, include_tail: bool,
                       adapters: AdapterBank | None = None, chunks_per_split: int = 0,
                       rec: torch.Tensor | None = None, corr: torch.Tensor | None = None):
        """Partial decode over quantized chunks [chunk_lo, chunk_hi) (+ the residual
        window and the correction when include_tail): returns (rec, corr) with
        rec fp32 [B, Hq, 4 + 2*128] = (m_log2, l, 0, 0, y_rot, y_raw) and corr fp32
        [B, Hq, 1 + 128] = (C_d, C_n) (zeros unless include_tail)."""
        q = q.to(self.device, torch.bfloat16).contiguous()
        if rec is None:
            rec = torch.empty((self.B, self.Hq, REC_FLOATS), dtype=torch.float32, device=self.device)
        if corr is None:
            corr = torch.zeros((self.B, self.Hq, CORR_FLOATS), dtype=torch.float32, device=self.device)
        o = self._opts(False, chunks_per_split)
        nbytes = _lib.load().kvlc_decode_workspace(ctypes.byref(self._struct), ctypes.byref(o))
        ws = self.decode_ws(nbytes)
        ad = _adapter_struct(adapters)
        _lib.call("kvlc_decode_partial", ctypes.byref(self._struct), ctypes.byref(ad), _ptr(q),
                  int(chunk_lo), int(chunk_hi), int(bool(include_tail)), _ptr(rec),
                  _ptr(corr) if include_tail else None, ctypes.byref(o), _ptr(ws), ws.numel(),
                  _lib.stream_handle())
        return rec, corr

    # ------------------------------------------------------------------ export
    def flush_due(self, adapters: AdapterBank | None = None) -> np.ndarray:
        """flush_group (cache.py:132-158) on every sequence whose window holds
        R + G tokens (deferred appends); returns the flushed sequence mask."""
        flush = self.res_len >= R + G
        if not np.any(flush):
            return flush
        if np.any(self.n_chunks + flush > self.max_chunks):
            raise ValueError(f"flush exceeds capacity of {self.max_tokens} tokens")
        f_c = (ctypes.c_int32 * self.B)(*flush.astype(np.int32).tolist())
        ws, nws = self._flush_ws(flush, adapters)
        _lib.call("kvlc_flush_due", ctypes.byref(self._struct), ctypes.byref(_adapter_struct(adapters)), f_c,
                  ws, nws, _lib.stream_handle())
        if _adapters_on(adapters):
            self.state_rank[flush] = RANK
        self.res_len = self.res_len - flush * G
        self.res_start = np.where(flush, (self.res_start + G) % SLOTS, self.res_start)
        self.n_chunks = self.n_chunks + flush
        return flush

    # ------------------------------------------------------------------ .kvlc I/O
    def serialize(self, b: int, kvh: int) -> bytes:
        """The reference's .kvlc bytes (serialize_cache, cache.py:209-230) of the
        per-head cache (b, kvh), written on the device in one kernel."""
        n, start, n_res, rank = (int(self.n_chunks[b]), int(self.res_start[b]), int(self.res_len[b]),
                                 int(self.state_rank[b]))
        lib = _lib.load()
        img = torch.empty(lib.kvlc_unit_image_bytes(n, n_res, rank), dtype=torch.uint8, device=self.device)
        _lib.call("kvlc_serialize_unit", ctypes.byref(self._struct), b * self.Hkv + kvh, n, start, n_res, rank,
                  _ptr(img), _lib.stream_handle())
        return img.cpu().numpy().tobytes()

    def load(self, b: int, images) -> None:
        """Load sequence b from one .kvlc image per kv head (deserialize_cache,
        cache.py:252-307).  The images must describe the serving format (d = G =
        R = 128, 2 bits, rotated values, rank 0 or 256) and agree on their token
        counts; the residual is stored at bf16 (the serving window precision)."""
        if len(images) != self.Hkv:
            raise ValueError(f"need {self.Hkv} images (one per kv head), got {len(images)}")
        hdrs = [fmt.parse_header(im) for im in images]
        for im, h in zip(images, hdrs):
            fmt.split(im, h)  # truncation / trailing-byte checks
            want = (D, G, R, 2, 1)
            got = (h.head_dim, h.group, h.window, h.bits, h.rotated)
            if got != want:
                raise ValueError(f"cache format (head_dim, group_size, residual_window, bits, rotated) = {got}; "
                                 f"the serving cache holds {want}")
            if h.rank not in (0, RANK):
                raise ValueError(f"adapter rank {h.rank} != cache state rank {RANK}")
        if len({(h.n_q, h.n_res, h.rank) for h in hdrs}) != 1:
            raise ValueError("kv-head images of one sequence disagree on token counts or state rank")
        h = hdrs[0]
        n = h.n_q // G
        if n > self.max_chunks or h.n_res > SLOTS:
            raise ValueError(f"cache of {h.n_q + h.n_res} tokens exceeds capacity of {self.max_tokens} tokens")
        for kvh, im in enumerate(images):
            dev = torch.frombuffer(bytearray(im), dtype=torch.uint8).to(self.device)
            _lib.call("kvlc_deserialize_unit", ctypes.byref(self._struct), b * self.Hkv + kvh, _ptr(dev), n,
                      h.n_res, h.rank, _lib.stream_handle())
        self.n_chunks[b], self.res_start[b], self.res_len[b], self.state_rank[b] = n, 0, h.n_res, h.rank

    def export_chunk(self, b: int, kvh: int, chunk: int) -> dict:
        """One quantized chunk in the reference layout (channel-axis key words
        (8, 128), value_rows words (128, 8), fp16 metadata)."""
        u = b * self.Hkv + kvh
        dev = self.device
        kw = torch.empty((8, 128), dtype=torch.int32, device=dev)
        vw = torch.empty((128, 8), dtype=torch.int32, device=dev)
        meta = torch.empty((4, 128), dtype=torch.float16, device=dev)
        _lib.call("kvlc_export_chunk", ctypes.byref(self._struct), u, chunk, _ptr(kw), _ptr(vw),
                  _ptr(meta[0]), _ptr(meta[1]), _ptr(meta[2]), _ptr(meta[3]), _lib.stream_handle())
        m = meta.cpu().numpy()
        return dict(kwords=kw.cpu().numpy().view(np.uint32), vwords=vw.cpu().numpy().view(np.uint32),
                    kscale=m[0], kzero=m[1], vscale=m[2], vzero=m[3])

    def export_unit(self, b: int, kvh: int, n_chunks: int | None = None) -> dict:
        """Every quantized chunk of one unit in the reference layout, stacked on a leading
        chunk axis (kvlc_export_chunk per chunk into device buffers, one host copy)."""
        u = b * self.Hkv + kvh
        n = int(self.n_chunks[b]) if n_chunks is None else n_chunks
        dev = self.device
        kw = torch.empty((n, 8, 128), dtype=torch.int32, device=dev)
        vw = torch.empty((n, 128, 8), dtype=torch.int32, device=dev)
        meta = torch.empty((n, 4, 128), dtype=torch.float16, device=dev)
        for ci in range(n):
            _lib.call("kvlc_export_chunk", ctypes.byref(self._struct), u, ci, _ptr(kw[ci]), _ptr(vw[ci]),
                      _ptr(meta[ci, 0]), _ptr(meta[ci, 1]), _ptr(meta[ci, 2]), _ptr(meta[ci, 3]),
                      _lib.stream_handle())
        m = meta.cpu().numpy()
        return dict(kwords=kw.cpu().numpy().view(np.uint32), vwords=vw.cpu().numpy().view(np.uint32),
                    kscale=m[:, 0], kzero=m[:, 1], vscale=m[:, 2], vzero=m[:, 3])

    def residual(self, b: int, kvh: int):
        """Live residual window of one unit, oldest first, as float32 host arrays."""
        u = b * self.Hkv + kvh
        start, n = int(self.res_start[b]), int(self.res_len[b])
        slots = [(start + i) % SLOTS for i in range(n)]
        k = self.kres[u].float().cpu().numpy()[slots]
        v = self.vres[u].float().cpu().numpy()[:, slots].T
        return k, v


def merge_records(recs: torch.Tensor, corr: torch.Tensor | None, literal: bool = False,
                  out: torch.Tensor | None = None, out_dtype: torch.dtype = torch.bfloat16) -> torch.Tensor:
    """LSE-merge n records [n, B, Hq, 4 + 2*128] (+ correction [B, Hq, 129])
    into out bf16 [B, Hq, 128] (`kvlc_merge_records`)."""
    n, B, Hq, width = recs.shape
    if width != REC_FLOATS:
        raise ValueError(f"record width {width} != {REC_FLOATS}")
    recs = recs.contiguous()
    if out is None:
        out = torch.empty((B, Hq, D), dtype=out_dtype, device=recs.device)
    _lib.call("kvlc_merge_records", _ptr(recs), n, B * Hq * REC_FLOATS,
              _ptr(corr.contiguous()) if corr is not None else None, B, Hq, int(bool(literal)),
              int(out.dtype == torch.float32), _ptr(out), _lib.stream_handle())
    return out
