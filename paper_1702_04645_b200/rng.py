"""Counter-based acceptance coin (rng.py of the reference), evaluated on the device."""

from __future__ import annotations

import numpy as np

__all__ = ["uniform01"]


def uniform01(seed: int, parts: tuple, ids) -> np.ndarray:
    """rng.py:34-43 for parts = (level, sweep): SplitMix64-keyed uniform [0, 1) per id."""
    if len(parts) != 2:
        raise ValueError("the device coin is keyed by (level, sweep)")
    from .forest import _scratch_ctx
    return _scratch_ctx(0).uniform01(seed, parts[0], parts[1], np.asarray(ids, dtype=np.int64))
