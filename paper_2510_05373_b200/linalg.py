"""Dense substrate of the reference package (quantkv.linalg, linalg.py:1-60) on the device.

`matmul` is a float64 cuBLAS GEMM, `softmax_rows` the max-shifted row softmax on CUDA
tensors; `rng` / `as_matrix` are the reference's host helpers.  Same names,
arguments and ValueError messages as the reference.
"""
from __future__ import annotations

import numpy as np
import torch

from ._device import device
from .adapter import rng  # noqa: F401  (PCG64, linalg.py:16-18)

Matrix = np.ndarray


def as_matrix(x, name: str = "matrix") -> Matrix:
    """linalg.py:21-25."""
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {a.shape}")
    return np.ascontiguousarray(a)


def matmul(a, b) -> Matrix:
    """linalg.py:28-35: a @ b with the reference's shape checks."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.ndim != 2 or b.ndim != 2:
        raise ValueError(f"matmul needs 2-D operands, got {a.shape} and {b.shape}")
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"cannot multiply {a.shape} by {b.shape}: inner dims differ")
    dt = np.result_type(a.dtype, b.dtype, np.float32)
    ta = torch.as_tensor(np.ascontiguousarray(a, dt), device=device())
    tb = torch.as_tensor(np.ascontiguousarray(b, dt), device=device())
    return (ta @ tb).cpu().numpy()


def softmax_rows(x) -> Matrix:
    """linalg.py:38-47: row-wise softmax with the max shift; -inf entries get weight 0."""
    t = torch.as_tensor(np.asarray(x, dtype=np.float64), device=device())
    e = torch.exp(t - t.max(dim=-1, keepdim=True).values)
    return (e / e.sum(dim=-1, keepdim=True)).cpu().numpy()
