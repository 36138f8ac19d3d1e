"""Drop-in correction-adapter feature maps (quantkv.adapter, adapter.py:38-101).

`CorrectionAdapter` holds the four (d, D/2) weights exactly like the
reference (same PCG64 initialisation, adapter.py:67-77); the feature map
phi(x) = [softmax(x W1), softmax(x W2)] runs in the `kvlc_ref_feature_map`
kernel (float64).  Adapter training and the .kvla format (adapter.py:104-362) are in
`train.py`.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import empty_dev, to_dev, to_host

WEIGHT_NAMES = ("w1_q", "w2_q", "w1_k", "w2_k")


def rng(seed: int) -> np.random.Generator:
    """Seeded generator with a fixed algorithm (PCG64), linalg.py:16-18."""
    return np.random.Generator(np.random.PCG64(seed))


@dataclass
class CorrectionAdapter:
    w1_q: np.ndarray
    w2_q: np.ndarray
    w1_k: np.ndarray
    w2_k: np.ndarray
    enabled: bool = True

    def __post_init__(self):
        shapes = {name: getattr(self, name).shape for name in WEIGHT_NAMES}
        first = shapes["w1_q"]
        if any(s != first for s in shapes.values()):
            raise ValueError(f"weight shapes must agree, got {shapes}")
        if len(first) != 2:
            raise ValueError(f"weights must be matrices, got shape {first}")

    @property
    def head_dim(self) -> int:
        return self.w1_q.shape[0]

    @property
    def rank(self) -> int:
        """Feature dimension D (each softmax half has D/2 entries)."""
        return 2 * self.w1_q.shape[1]

    def weights(self) -> dict:
        return {name: getattr(self, name) for name in WEIGHT_NAMES}

    @classmethod
    def initialize(cls, head_dim: int, rank: int, seed: int = 0, init_scale: float = 1.0,
                   enabled: bool = True) -> "CorrectionAdapter":
        """Fresh adapter with N(0, (init_scale/sqrt(d))^2) weights."""
        if rank < 2 or rank % 2:
            raise ValueError(f"rank must be an even integer >= 2, got {rank}")
        if head_dim < 1:
            raise ValueError(f"head_dim must be >= 1, got {head_dim}")
        g = rng(seed)
        std = init_scale / np.sqrt(head_dim)
        mats = [g.standard_normal((head_dim, rank // 2)) * std for _ in range(4)]
        return cls(*mats, enabled=enabled)

    def device_weights(self):
        """float64 device copies (w1_q, w2_q, w1_k, w2_k)."""
        return tuple(to_dev(np.ascontiguousarray(getattr(self, n), np.float64)) for n in WEIGHT_NAMES)


def _feature_map_dev(d_x, n: int, d: int, d_w1, d_w2, h: int):
    d_out = empty_dev((n, 2 * h), "f64")
    _lib.call("kvlc_ref_feature_map", _lib.ptr(d_x), n, d, _lib.ptr(d_w1), _lib.ptr(d_w2), h,
              _lib.ptr(d_out), _lib.stream_handle())
    return d_out


def feature_map(x, w1: np.ndarray, w2: np.ndarray) -> np.ndarray:
    """Two-softmax feature map of one vector or a stack of rows (adapter.py:80-88)."""
    x = np.asarray(x, dtype=np.float64)
    single = x.ndim == 1
    rows = x[np.newaxis, :] if single else x
    if rows.shape[1] != w1.shape[0]:
        raise ValueError(f"feature input dim {rows.shape[1]} != weight dim {w1.shape[0]}")
    h = w1.shape[1]
    out = to_host(_feature_map_dev(to_dev(rows), rows.shape[0], rows.shape[1],
                                   to_dev(np.asarray(w1, np.float64)),
                                   to_dev(np.asarray(w2, np.float64)), h), "f64")
    return out[0] if single else out


def phi_q(adapter: CorrectionAdapter, x) -> np.ndarray:
    return feature_map(x, adapter.w1_q, adapter.w2_q)


def phi_k(adapter: CorrectionAdapter, x) -> np.ndarray:
    return feature_map(x, adapter.w1_k, adapter.w2_k)


def correction_term(q, k_err, adapter: CorrectionAdapter) -> float:
    """f(q, k_err) = phi_q(q) . phi_k(k_err) (adapter.py:99-101)."""
    return float(phi_q(adapter, q) @ phi_k(adapter, k_err))
