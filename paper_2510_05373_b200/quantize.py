"""Drop-in `quantkv.quantize` API backed by libkvlinc (sm_100a).

Same names, arguments, return types and ValueError messages as the
reference module (/root/reference/pkg/src/quantkv/quantize.py); the
arithmetic runs in the CUDA kernels `kvlc_ref_quantize`, `kvlc_ref_pack`,
`kvlc_ref_unpack` and `kvlc_ref_dequantize` (float64, bit-exact codes).
Host arrays in, host arrays out, as in the reference.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import to_dev, to_host, empty_dev

AXES = ("channel", "token")                 # quantize.py:29
ROTATIONS = ("none", "pre", "post")         # quantize.py:30
QUANT_BITS = (2, 3, 4, 8)                   # quantize.py:33
_LANE_BITS = {2: 2, 3: 4, 4: 4, 8: 8}       # quantize.py:37


@dataclass(frozen=True)
class QuantConfig:
    """How one tensor is grouped, rotated and quantized (quantize.py:40-64)."""

    bits: int = 2
    group_size: int = 128
    axis: str = "token"
    rotation: str = "none"

    def __post_init__(self):
        if self.bits not in QUANT_BITS + (16,):
            raise ValueError(f"bits must be one of {QUANT_BITS + (16,)}, got {self.bits}")
        if self.group_size < 1:
            raise ValueError(f"group_size must be >= 1, got {self.group_size}")
        if self.axis not in AXES:
            raise ValueError(f"axis must be one of {AXES}, got {self.axis!r}")
        if self.rotation not in ROTATIONS:
            raise ValueError(f"rotation must be one of {ROTATIONS}, got {self.rotation!r}")

    @property
    def is_passthrough(self) -> bool:
        return self.bits == 16

    def label(self) -> str:
        return f"{self.axis}/{self.rotation}"


def _lanes(bits: int) -> int:
    return 32 // _LANE_BITS[bits]


def pack_codes(codes, bits: int) -> np.ndarray:
    """Pack integer codes into little-endian lanes of uint32 words (quantize.py:71-94)."""
    if bits not in _LANE_BITS:
        raise ValueError(f"cannot pack {bits}-bit codes, supported: {sorted(_LANE_BITS)}")
    codes = np.asarray(codes)
    if codes.ndim not in (1, 2):
        raise ValueError(f"codes must be 1-D or 2-D, got shape {codes.shape}")
    if codes.size and (codes.min() < 0 or codes.max() > (1 << bits) - 1):
        raise ValueError(f"codes out of range for {bits} bits")
    rows, n = (1, codes.shape[0]) if codes.ndim == 1 else codes.shape
    nwords = -(-n // _lanes(bits)) if n else 0
    if rows * nwords == 0:
        out = np.zeros((rows, nwords), np.uint32)
        return out[0] if codes.ndim == 1 else out
    d_codes = to_dev(np.ascontiguousarray(codes.reshape(rows, n), dtype=np.uint8))
    d_words = empty_dev((rows, nwords), "u32")
    _lib.call("kvlc_ref_pack", _lib.ptr(d_codes), rows, n, bits, _lib.ptr(d_words), _lib.stream_handle())
    out = to_host(d_words, "u32")
    return out[0] if codes.ndim == 1 else out


def unpack_codes(words, count: int, bits: int) -> np.ndarray:
    """Inverse of pack_codes (quantize.py:97-114)."""
    if bits not in _LANE_BITS:
        raise ValueError(f"cannot unpack {bits}-bit codes, supported: {sorted(_LANE_BITS)}")
    words = np.asarray(words, dtype=np.uint32)
    if words.ndim not in (1, 2):
        raise ValueError(f"words must be 1-D or 2-D, got shape {words.shape}")
    one_d = words.ndim == 1
    w = words.reshape(1, -1) if one_d else words
    if count > w.shape[1] * _lanes(bits):
        raise ValueError(f"count {count} exceeds capacity of {w.shape[1]} words")
    if w.shape[0] * count == 0:
        out = np.zeros((w.shape[0], count), np.uint8)
        return out[0] if one_d else out
    d_words = to_dev(np.ascontiguousarray(w))
    d_codes = empty_dev((w.shape[0], count), "u8")
    _lib.call("kvlc_ref_unpack", _lib.ptr(d_words), w.shape[0], w.shape[1], count, bits,
              _lib.ptr(d_codes), _lib.stream_handle())
    out = to_host(d_codes, "u8")
    return out[0] if one_d else out


def _quantize_dev(d_x, rows: int, cols: int, bits: int, group: int, axis: int):
    """Device quantization: returns device (words, scales, zeros)."""
    lanes = _lanes(bits)
    if axis == _lib.AXIS_TOKEN:
        wshape, mshape = (rows, -(-cols // lanes)), (rows, -(-cols // group))
    else:
        wshape, mshape = (-(-rows // lanes), cols), (-(-rows // group), cols)
    d_words = empty_dev(wshape, "u32")
    d_scales = empty_dev(mshape, "f64")
    d_zeros = empty_dev(mshape, "f64")
    scratch = empty_dev((rows * cols,), "u8")
    _lib.call("kvlc_ref_quantize", _lib.ptr(d_x), rows, cols, bits, group, axis, _lib.ptr(d_words),
              _lib.ptr(d_scales), _lib.ptr(d_zeros), _lib.ptr(scratch), _lib.stream_handle())
    return d_words, d_scales, d_zeros


def quantize_group(values, bits: int):
    """Quantize one 1-D group; returns (codes, scale, zero) (quantize.py:117-135)."""
    if bits not in QUANT_BITS:
        raise ValueError(f"bits must be one of {QUANT_BITS}, got {bits}")
    v = np.asarray(values, dtype=np.float64)
    if v.ndim != 1 or v.size == 0:
        raise ValueError(f"group must be a non-empty 1-D array, got shape {v.shape}")
    d_words, d_s, d_z = _quantize_dev(to_dev(v.reshape(1, -1)), 1, v.size, bits, v.size, _lib.AXIS_TOKEN)
    codes = unpack_codes(to_host(d_words, "u32"), v.size, bits)[0]
    return codes, float(to_host(d_s, "f64")[0, 0]), float(to_host(d_z, "f64")[0, 0])


def dequantize_group(codes, scale: float, zero: float) -> np.ndarray:
    """scale * codes + zero in float64 (quantize.py:138-144)."""
    codes = np.asarray(codes)
    if codes.size and (codes.min() < 0):
        raise ValueError("codes must be unsigned")
    if scale < 0:
        raise ValueError(f"scale must be >= 0, got {scale}")
    if codes.size == 0:
        return np.zeros(codes.shape)
    if codes.max() > 255:
        raise ValueError("codes out of range for 8 bits")
    flat = codes.reshape(1, -1)
    # keep every device temporary referenced until the launch is queued
    d_words = to_dev(pack_codes(flat.astype(np.uint8), 8))
    d_scale = to_dev(np.array([[scale]], dtype=np.float64))
    d_zero = to_dev(np.array([[zero]], dtype=np.float64))
    d_out = empty_dev(flat.shape, "f64")
    _lib.call("kvlc_ref_dequantize", _lib.ptr(d_words), _lib.ptr(d_scale), _lib.ptr(d_zero), 1,
              flat.shape[1], 8, flat.shape[1], _lib.AXIS_TOKEN, _lib.ptr(d_out), _lib.stream_handle())
    return to_host(d_out, "f64").reshape(codes.shape)


def expected_quant_mse(scale: float) -> float:
    """Uniform-error model of round-to-nearest: scale^2 / 12 (quantize.py:147-151)."""
    if scale < 0:
        raise ValueError(f"scale must be >= 0, got {scale}")
    return scale * scale / 12.0


@dataclass
class QuantizedTensor:
    """Packed codes plus per-group metadata (quantize.py:154-180); host arrays.

    token:   codes (r, ceil(c/L)),  scales/zeros (r, ceil(c/G))
    channel: codes (ceil(r/L), c),  scales/zeros (ceil(r/G), c)
    """

    codes: np.ndarray
    scales: np.ndarray
    zeros: np.ndarray
    rows: int
    cols: int
    config: QuantConfig

    @property
    def group_count(self) -> int:
        return self.scales.size

    def dequantize(self) -> np.ndarray:
        cfg = self.config
        axis = _lib.AXIS_TOKEN if cfg.axis == "token" else _lib.AXIS_CHANNEL
        d_out = empty_dev((self.rows, self.cols), "f64")
        d_codes = to_dev(np.ascontiguousarray(self.codes, np.uint32))
        d_scales = to_dev(np.ascontiguousarray(self.scales, np.float64))
        d_zeros = to_dev(np.ascontiguousarray(self.zeros, np.float64))
        _lib.call("kvlc_ref_dequantize", _lib.ptr(d_codes), _lib.ptr(d_scales), _lib.ptr(d_zeros),
                  self.rows, self.cols, cfg.bits, cfg.group_size, axis, _lib.ptr(d_out),
                  _lib.stream_handle())
        return to_host(d_out, "f64")


def quantize_tensor(x, config: QuantConfig) -> QuantizedTensor:
    """Group-quantize a matrix along the configured axis (quantize.py:220-239)."""
    if config.is_passthrough:
        raise ValueError("bits=16 is a passthrough config; nothing to quantize")
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2 or x.size == 0:
        raise ValueError(f"expected a non-empty matrix, got shape {x.shape}")
    d_x = to_dev(np.ascontiguousarray(x))
    from ._device import all_finite
    if not all_finite(d_x):
        raise ValueError("matrix contains non-finite entries")
    axis = _lib.AXIS_TOKEN if config.axis == "token" else _lib.AXIS_CHANNEL
    d_w, d_s, d_z = _quantize_dev(d_x, x.shape[0], x.shape[1], config.bits, config.group_size, axis)
    return QuantizedTensor(to_host(d_w, "u32"), to_host(d_s, "f64"), to_host(d_z, "f64"),
                           x.shape[0], x.shape[1], config)
