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

import ctypes

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


class RecoveryPipeline:
    """Double-buffered multi-stream serving loop for one modality.

    A server hosting ``n`` conference streams of one resolution receives, per
    frame time, each stream's decoded corrupted plane and its P-frame shard
    state.  ``submit`` stages them (pinned host memory), then enqueues

      copy stream     H2D of the planes + loss-mask jobs into buffer i
      compute stream  nvrec_loss_mask -> nvrec_recover_u8 (device-resident
                      reference rings) -> ring push of the recovered planes
      copy stream     D2H of the recovered planes

    with buffer i = step % 2, so step t's transfers overlap step t-1's
    compute.  ``result(handle)`` waits for that step's D2H and returns the
    pinned host array (b, h, w, c).  The rings start from ``init_refs``
    (device u8 (n, k, h, w, c)); every recovered plane becomes the newest
    reference of its stream (reference receiver.py:268-269)."""

    def __init__(self, engine: RecoveryEngine, n: int, h: int, w: int,
                 shard_len: int, max_header: int, max_shards: int, init_refs: torch.Tensor):
        from .lossmask import LossMaskBatch
        self.engine = engine
        self.n, self.h, self.w = n, h, w
        self.c = engine.channels
        cfg = engine.model.config
        self.k, self.F = cfg.k, cfg.stack_len
        dev = init_refs.device
        self.device = dev
        # slots per stream: k ring entries + 2 corrupted-plane buffers
        self.S = self.k + 2
        self.frames = torch.empty((n, self.S, h, w, self.c), dtype=torch.uint8, device=dev)
        self.frames[:, :self.k].copy_(init_refs)
        self.flat = self.frames.view(n * self.S, h, w, self.c)
        self.head = [0] * n                      # ring position of the oldest reference
        self.nblk = (h // 16) * (w // 16)
        self.lm = [LossMaskBatch(n, max_header, max_shards, self.nblk, 1, dev) for _ in range(2)]
        self.out = [torch.empty((n, h, w, self.c), dtype=torch.uint8, device=dev)
                    for _ in range(2)]
        self.host_in = [torch.empty((n, h, w, self.c), dtype=torch.uint8).pin_memory()
                        for _ in range(2)]
        self.host_out = [torch.empty((n, h, w, self.c), dtype=torch.uint8).pin_memory()
                         for _ in range(2)]
        self.index = [torch.empty((n, self.F), dtype=torch.int32).pin_memory() for _ in range(2)]
        self.dev_index = [torch.empty((n, self.F), dtype=torch.int32, device=dev)
                          for _ in range(2)]
        self.s_h2d = torch.cuda.Stream(dev)
        self.s_cmp = torch.cuda.Stream(dev)
        self.s_d2h = torch.cuda.Stream(dev)
        self.ev_h2d = [torch.cuda.Event() for _ in range(2)]
        self.ev_cmp = [torch.cuda.Event() for _ in range(2)]
        self.ev_d2h = [torch.cuda.Event() for _ in range(2)]
        self.step = 0
        self.shard_len = shard_len

    def h2d_bytes(self) -> int:
        return int(self.host_in[0].numel() + self.lm[0].h2d_bytes + self.index[0].numel() * 4)

    def d2h_bytes(self) -> int:
        return int(self.host_out[0].numel())

    def submit(self, planes: np.ndarray | None, frames) -> int:
        """planes: (n, h, w, c) u8 host array (or None if already written into
        ``host_in[step % 2]``); frames: n ``PFrameShards``.  Returns a handle."""
        i = self.step & 1
        if self.step >= 2:
            self.ev_h2d[i].synchronize()          # staging buffers of step-2 are free
            self.ev_d2h[i].synchronize()          # host_out[i] consumed by the caller
        if planes is not None:
            self.host_in[i].numpy()[...] = planes
        self.lm[i].stage(frames)
        idx = self.index[i].numpy()
        for s in range(self.n):
            ring = [(self.head[s] + j) % self.k for j in range(self.k)]
            idx[s] = [s * self.S + r for r in ring] + [s * self.S + self.k + i]
        # H2D: plane into its buffer slot, loss-mask jobs, slot table
        self.s_h2d.wait_event(self.ev_cmp[i]) if self.step >= 2 else None
        with torch.cuda.stream(self.s_h2d):
            self.frames[:, self.k + i].copy_(self.host_in[i], non_blocking=True)
            self.lm[i].dev_in.copy_(self.lm[i].host, non_blocking=True)
            self.dev_index[i].copy_(self.index[i], non_blocking=True)
            self.ev_h2d[i].record(self.s_h2d)
        # compute
        self.s_cmp.wait_event(self.ev_h2d[i])
        with torch.cuda.stream(self.s_cmp):
            lib = self.lm[i].lib
            _native.check(lib.nvrec_loss_mask(ctypes.c_void_p(self.lm[i].dev_in.data_ptr()),
                                              self.lm[i].n,
                                              ctypes.c_void_p(int(self.s_cmp.cuda_stream))))
            if self.step >= 2:
                self.s_cmp.wait_event(self.ev_d2h[i])   # out[i] drained
            self.engine.recover_device(self.flat, self.dev_index[i], self.lm[i].wire,
                                       self.out[i])
            # ring push: the recovered plane replaces each stream's oldest ref
            for s in range(self.n):
                self.frames[s, self.head[s]].copy_(self.out[i][s], non_blocking=True)
            self.ev_cmp[i].record(self.s_cmp)
        for s in range(self.n):
            self.head[s] = (self.head[s] + 1) % self.k
        # D2H
        self.s_d2h.wait_event(self.ev_cmp[i])
        with torch.cuda.stream(self.s_d2h):
            self.host_out[i].copy_(self.out[i], non_blocking=True)
            self.ev_d2h[i].record(self.s_d2h)
        self.step += 1
        return i

    def result(self, handle: int) -> np.ndarray:
        self.ev_d2h[handle].synchronize()
        return self.host_out[handle].numpy()


def recover_depth16(model, plane: np.ndarray, grid: np.ndarray, refs: list) -> np.ndarray:
    """16-bit depth extension of ``_recover`` (SPEC.md:74 calls 16-bit depth
    an extension point; the reference codec and wire format are u8-only).

    Planes are u16 (h, w); the float module API is fed ``u16 / 65535`` (the
    16-bit analogue of server.py:189), the output is quantised with
    ``clip(out * 65535 + 0.5, 0, 65535)`` and merged through the block mask.
    Use a ``precision="precise"`` model: it keeps the error below 1/65535 of
    full scale (the north_star's <= 1 mm at 1 mm per depth unit)."""
    if not refs or not np.asarray(grid).any():
        return np.ascontiguousarray(plane)
    cfg = model.config
    dev = _native.require_cuda()
    refs = list(refs)[-cfg.k:]
    host = np.stack(refs + [plane]).astype(np.uint16)
    stack = torch.from_numpy(host.astype(np.int32)).to(dev).float().div_(65535.0)[None, :, None]
    pix = np.repeat(np.repeat(np.asarray(grid, bool), MASK_BLOCK, 0), MASK_BLOCK, 1)
    mask = torch.from_numpy(pix).to(dev)[None]
    out = model(stack, mask)[0, 0]
    q = torch.clamp(out * 65535.0 + 0.5, 0, 65535).to(torch.int32).cpu().numpy().astype(np.uint16)
    return np.where(pix, q, plane)
