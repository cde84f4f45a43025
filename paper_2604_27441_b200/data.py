"""Constants and the synthetic block mask of ``nvrec.data``
(``pkg/nvrec/src/nvrec/data.py:26-28,137-142``).  Corpus I/O (training
data) is out of scope for the recovery path."""

from __future__ import annotations

import numpy as np

MOD_RGB = 0
MOD_DEPTH = 1
MASK_BLOCK = 16


def synthetic_mask(height: int, width: int, ratio: float,
                   rng: np.random.Generator) -> np.ndarray:
    """Per-pixel bool mask made of whole 16-px blocks, ~``ratio`` of them set
    (same draw order as data.py:137-142, so seeds reproduce)."""
    grid = rng.random((height // MASK_BLOCK, width // MASK_BLOCK)) < ratio
    return np.repeat(np.repeat(grid, MASK_BLOCK, 0), MASK_BLOCK, 1)
