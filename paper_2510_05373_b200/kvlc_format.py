"""The `.kvlc` per-head cache file format (quantkv cache.py:197-307).

Little-endian: magic "KVLC", nine u32 (version, head_dim, adapter_rank, group_size,
residual_window, bits, values_rotated, quantized_tokens, residual_len), then
  key chunk codes    u32 [chunks][ceil(G/L)][d]
  value codes        u32 [n_q][ceil(d/L)]
  key scales, zeros  f16 [1][d] each, per chunk (scales then zeros)
  value scales       f16 [n_q][ceil(d/G)], then value zeros
  residual keys      f16 [n_res][d], then residual values
  S f16 [d][rank], then P f16 [rank]  (only when rank > 0)
The 16-bit fields make the file lossy by design (cache.py:203-204).

Header / section validation raises `CacheFormatError` with the reference's
messages ("bad magic at byte 0", "unsupported cache version", "truncated cache
file at byte", "trailing bytes at byte").  The per-head shim
(`cache.serialize_cache`) and the batched serving cache
(`BatchedKVCache.serialize` / `.load`) both use this module; the serving cache
writes and reads the byte image on the device (`kvlc_serialize_unit`).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

MAGIC = b"KVLC"          # cache.py:31
VERSION = 1              # cache.py:32
HEADER = struct.Struct("<4s9I")
_LANE_BITS = {2: 2, 3: 4, 4: 4, 8: 8}


class CacheFormatError(ValueError):
    """Malformed .kvlc data (cache.py:233-234)."""


@dataclass(frozen=True)
class Header:
    version: int
    head_dim: int
    rank: int
    group: int
    window: int
    bits: int
    rotated: int
    n_q: int
    n_res: int

    def pack(self) -> bytes:
        return HEADER.pack(MAGIC, self.version, self.head_dim, self.rank, self.group, self.window,
                           self.bits, self.rotated, self.n_q, self.n_res)

    def sections(self):
        """(name, dtype, shape) of every section after the header, in file order."""
        d, g = self.head_dim, self.group
        lanes = 32 // _LANE_BITS[self.bits]
        kw, vw, vg = -(-g // lanes), -(-d // lanes), -(-d // g)
        chunks = self.n_q // g
        out = [("kcodes", "<u4", (chunks, kw, d)), ("vcodes", "<u4", (self.n_q, vw)),
               ("kmeta", "<f2", (chunks, 2, 1, d)), ("vscales", "<f2", (self.n_q, vg)),
               ("vzeros", "<f2", (self.n_q, vg)), ("res_k", "<f2", (self.n_res, d)),
               ("res_v", "<f2", (self.n_res, d))]
        if self.rank:
            out += [("s", "<f2", (d, self.rank)), ("p", "<f2", (self.rank,))]
        return out

    def nbytes(self) -> int:
        return HEADER.size + sum(int(np.prod(s)) * np.dtype(t).itemsize for _, t, s in self.sections())


def parse_header(data: bytes) -> Header:
    """Magic and version checks of deserialize_cache (cache.py:252-257)."""
    if bytes(data[:4]) != MAGIC:
        raise CacheFormatError(f"bad magic at byte 0: {bytes(data[:4])!r}")
    if len(data) < HEADER.size:
        raise CacheFormatError(f"truncated cache file at byte 4: need {HEADER.size - 4} more bytes")
    _, version, d, rank, g, r, bits, rotated, n_q, n_res = HEADER.unpack_from(data)
    if version != VERSION:
        raise CacheFormatError(f"unsupported cache version {version} at byte 4")
    if bits not in _LANE_BITS:
        raise CacheFormatError(f"bits must be one of (2, 3, 4, 8), got {bits}")
    return Header(version, d, rank, g, r, bits, rotated, n_q, n_res)


def split(data: bytes, h: Header) -> dict:
    """Sections as numpy arrays (views into `data`), with the reader's
    truncation and trailing-byte checks (cache.py:237-249, 303-304)."""
    off, out = HEADER.size, {}
    for name, dt, shape in h.sections():
        n = int(np.prod(shape)) * np.dtype(dt).itemsize
        if off + n > len(data):
            raise CacheFormatError(f"truncated cache file at byte {off}: need {n} more bytes")
        out[name] = np.frombuffer(data, dtype=dt, count=int(np.prod(shape)), offset=off).reshape(shape)
        off += n
    if off != len(data):
        raise CacheFormatError(f"trailing bytes at byte {off}")
    return out


def join(h: Header, parts: dict) -> bytes:
    """Header + sections in file order (cache.py:209-230)."""
    out = [h.pack()]
    for name, dt, shape in h.sections():
        a = np.ascontiguousarray(np.asarray(parts[name]).astype(dt, copy=False)).reshape(shape)
        out.append(a.tobytes())
    return b"".join(out)
