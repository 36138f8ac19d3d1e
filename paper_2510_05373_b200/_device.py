"""Device-memory plumbing (torch tensors as allocations, H2D/D2H copies).

torch is only the allocator / copy engine / stream provider here; every
computation on the hot path is a libkvlinc kernel.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib

_KINDS = {
    "u8": (torch.uint8, np.uint8),
    "u32": (torch.int32, np.uint32),   # raw 32-bit words; viewed as uint32 on the host
    "i32": (torch.int32, np.int32),
    "u16": (torch.int16, np.uint16),   # raw 16-bit storage (f16 / bf16 bit patterns)
    "f32": (torch.float32, np.float32),
    "f64": (torch.float64, np.float64),
}


def device() -> torch.device:
    _lib.require_device()
    return torch.device("cuda", torch.cuda.current_device())


def empty_dev(shape, kind: str) -> torch.Tensor:
    return torch.empty(tuple(shape), dtype=_KINDS[kind][0], device=device())


def zeros_dev(shape, kind: str) -> torch.Tensor:
    return torch.zeros(tuple(shape), dtype=_KINDS[kind][0], device=device())


def to_dev(a: np.ndarray) -> torch.Tensor:
    """Copy a host array to the device, preserving bits (uint32 -> int32 storage)."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    elif a.dtype == np.uint16:
        a = a.view(np.int16)
    return torch.from_numpy(a).to(device(), non_blocking=False)


def to_host(t: torch.Tensor, kind: str) -> np.ndarray:
    out = t.detach().cpu().numpy()
    want = _KINDS[kind][1]
    if out.dtype != want:
        out = out.view(want)
    return out


def all_finite(t: torch.Tensor) -> bool:
    return bool(torch.isfinite(t).all().item())
