"""Host-side array helpers on the drop-in path (reference arrays.py:54-67)."""

from __future__ import annotations

import numpy as np

from .errors import ShapeError

__all__ = ["mask_apply"]


def mask_apply(x, mask):
    """Zero ``x`` where ``mask`` is 0; observed entries are copied bit-exactly."""
    x = np.asarray(x)
    mask = np.asarray(mask)
    if x.shape != mask.shape:
        raise ShapeError(f"mask shape {mask.shape} does not match tensor shape {x.shape}")
    out = np.zeros_like(x)
    on = mask == 1
    out[on] = x[on]
    return out
