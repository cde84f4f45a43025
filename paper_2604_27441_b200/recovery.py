"""Batched u8 recovery engine: the compute of ``RecoveryServer._recover``.

``_recover`` (reference server.py:181-196) stacks ``refs[-k:] + [plane]``,
normalises by 255, runs the model, quantises with
``clip(out*255+0.5, 0, 255).astype(u8)`` and merges through the block mask.
``RecoveryEngine`` does all of it in one ``nvrec_recover_u8`` call over a
batch of independent streams: u8 planes go to the device as they are (no
f32 staging), the mask stays a wire bitset, and only masked patches are
decoded (exact -- the merge discards the rest).

Frame staging: the engine owns a device slot buffer; each stream's stack
is described by an int32 slot table (oldest first, front-padded by repeating
the oldest slot, model.py:99-101), so a device-resident reference ring
(``DeviceRing``) needs no copies when it rotates.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .data import MASK_BLOCK


def pack_grid(grid: np.ndarray) -> np.ndarray:
    """Row-major MSB-first bitset of a bool block grid (recovery.py:221)."""
    return np.packbits(np.asarray(grid, dtype=bool).reshape(-1))


def stack_slots(n_refs: int, k: int, stack_len: int) -> list[int]:
    """Slot order of ``refs[-k:] + [plane]`` front-padded to ``stack_len``.

    Slots 0..n_refs-1 hold the references (oldest first), slot n_refs the
    corrupted plane (server.py:189, model.py:99-101)."""
    used = list(range(max(0, n_refs - k), n_refs)) + [n_refs]
    return [used[0]] * (stack_len - len(used)) + used


class RecoveryEngine:
    """Runs ``nvrec_recover_u8`` for one model (one modality) on one device."""

    def __init__(self, model, precision: str = "fast"):
        self.model = model
        self.precision = _native.precision_code(precision)

    @property
    def channels(self) -> int:
        return self.model.channels

    def recover_device(self, frames: torch.Tensor, frame_index: torch.Tensor,
                       mask_bits: torch.Tensor, out: torch.Tensor | None = None
                       ) -> torch.Tensor:
        """All-device batched call.

        frames: u8 (n_slots, h, w, c) on the device; frame_index: int32
        (b, stack_len) slot table; mask_bits: u8 (b, ceil(gh*gw/8)).
        Returns u8 (b, h, w, c) merged planes."""
        nat = self.model.native(frames.device)
        _, h, w, c = frames.shape
        b = frame_index.shape[0]
        if c != self.channels:
            raise ValueError("expected %d channels, got %d" % (self.channels, c))
        if out is None:
            out = torch.empty((b, h, w, c), dtype=torch.uint8, device=frames.device)
        return nat.recover_u8(frames, frame_index, mask_bits, out, b, h, w, self.precision)

    def recover(self, plane: np.ndarray, grid: np.ndarray, refs: list) -> np.ndarray:
        """Host-buffer call with ``_recover``'s signature and echo rules."""
        plane = np.asarray(plane)
        pl3 = plane if plane.ndim == 3 else plane[:, :, None]
        if not refs or not np.asarray(grid).any():
            return np.ascontiguousarray(plane)
        h, w, c = pl3.shape
        cfg = self.model.config
        dev = _native.require_cuda()
        refs = list(refs)[-cfg.k:]
        host = np.stack([np.asarray(r).reshape(h, w, c) for r in refs] + [pl3])
        slots = stack_slots(len(refs), cfg.k, cfg.stack_len)
        frames = torch.from_numpy(host).to(dev, non_blocking=True)
        index = torch.tensor([slots], dtype=torch.int32).to(dev, non_blocking=True)
        bits = torch.from_numpy(pack_grid(grid)[None]).to(dev, non_blocking=True)
        out = self.recover_device(frames, index, bits)
        res = out[0].cpu().numpy()
        return res if plane.ndim == 3 else res[:, :, 0]


def grid_shape(h: int, w: int) -> tuple[int, int]:
    return h // MASK_BLOCK, w // MASK_BLOCK
