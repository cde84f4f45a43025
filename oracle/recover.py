"""Oracle: restatement of ``RecoveryServer._recover`` and the wire mask.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Reference: ``pkg/nvrec/src/nvrec/server.py:150-196`` (request parse and
``_recover``) and ``pkg/src/rgbdstream/recovery.py:86-91,214-227`` (client
``masked_merge`` and ``encode_request``'s ``np.packbits`` mask).
"""

from __future__ import annotations

import numpy as np
import torch

from . import nvrec_forward

MASK_BLOCK = 16          # nvrec/data.py:28, rgbdstream/recovery.py:32


def grid_to_pixels(grid: np.ndarray) -> np.ndarray:
    """server.py:183 -- block grid -> per-pixel bool mask."""
    return np.repeat(np.repeat(grid, MASK_BLOCK, 0), MASK_BLOCK, 1)


def pack_grid(grid: np.ndarray) -> bytes:
    """recovery.py:221 -- row-major MSB-first bitset."""
    return np.packbits(np.asarray(grid, bool).reshape(-1)).tobytes()


def unpack_grid(bits, gh: int, gw: int) -> np.ndarray:
    """server.py:166-168 -- inverse of ``pack_grid``."""
    raw = np.frombuffer(bytes(bits), np.uint8, (gh * gw + 7) // 8)
    return np.unpackbits(raw, count=gh * gw).astype(bool).reshape(gh, gw)


def recover(state: dict | None, arch: nvrec_forward.Arch, channels: int,
            plane: np.ndarray, grid: np.ndarray, refs: list[np.ndarray],
            echo: bool = False) -> np.ndarray:
    """server.py:181-196.  ``plane``/``refs`` are u8 (h, w, c); ``grid`` is
    the (h/16, w/16) bool block grid.  Returns the merged u8 (h, w, c)."""
    pix = grid_to_pixels(grid)                                    # :183
    if echo or state is None or not refs or not pix.any():       # :184-186
        return np.ascontiguousarray(plane)
    k = arch.k                                                    # :188
    stack_np = np.stack(list(refs[-k:]) + [plane]).astype(np.float32) / 255.0
    stack = torch.from_numpy(stack_np).permute(0, 3, 1, 2)[None]  # :189-190
    mask = torch.from_numpy(pix)[None]                            # :191
    out = nvrec_forward.forward(state, arch, channels, stack, mask)  # :192-193
    out = out[0].permute(1, 2, 0).numpy()
    pred = np.clip(out * 255.0 + 0.5, 0, 255).astype(np.uint8)   # :194
    return np.where(pix[:, :, None], pred, plane)                 # :196


def recover16(state: dict | None, arch: nvrec_forward.Arch, plane: np.ndarray,
              grid: np.ndarray, refs: list[np.ndarray]) -> np.ndarray:
    """16-bit depth extension of server.py:181-196 (SPEC.md:74 names 16-bit
    depth an extension point; the wire format is u8): the same stack / mask /
    forward / merge with 65535 in place of 255.  ``plane``/``refs`` are u16
    (h, w); returns the merged u16 (h, w)."""
    pix = grid_to_pixels(grid)
    if state is None or not refs or not pix.any():
        return np.ascontiguousarray(plane)
    stack_np = np.stack(list(refs[-arch.k:]) + [plane]).astype(np.float32) / 65535.0
    stack = torch.from_numpy(stack_np)[None, :, None]
    out = nvrec_forward.forward(state, arch, 1, stack, torch.from_numpy(pix)[None]).numpy()[0, 0]
    pred = np.clip(out * 65535.0 + 0.5, 0, 65535).astype(np.uint16)
    return np.where(pix, pred, plane)


def masked_merge(original: np.ndarray, recovered: np.ndarray,
                 grid: np.ndarray) -> np.ndarray:
    """recovery.py:86-91 (client-side re-merge)."""
    channels = 1 if original.ndim == 2 else original.shape[2]
    pix = grid_to_pixels(grid)
    if channels > 1:
        pix = np.repeat(pix[:, :, None], channels, axis=2)
    return np.where(pix, recovered, original)
