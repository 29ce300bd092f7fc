"""Counter-based acceptance coin (rng.py of the reference), evaluated on the device."""

from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["uniform01"]

_ctx = {}


def uniform01(seed: int, parts: tuple, ids) -> np.ndarray:
    """rng.py:34-43 for parts = (level, sweep): SplitMix64-keyed uniform [0, 1) per id."""
    if len(parts) != 2:
        raise ValueError("the device coin is keyed by (level, sweep)")
    if "c" not in _ctx:
        _ctx["c"] = _lib.Context(0)
    return _ctx["c"].uniform01(seed, parts[0], parts[1], np.asarray(ids, dtype=np.int64))
