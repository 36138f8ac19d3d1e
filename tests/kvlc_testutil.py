"""Small helpers shared by the tests (kept out of conftest so they import by name)."""
import numpy as np


def bf16_round(x):
    """fp32 -> bf16 (round to nearest even) -> float64, as the serving inputs are."""
    f = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((f + 0x7FFF + ((f >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)
