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
                       mask_bits: torch.Tensor, out: torch.Tensor | None = None,
                       in_place: bool = False, native=None) -> torch.Tensor | None:
        """All-device batched call.

        frames: u8 (n_slots, h, w, c) on the device; frame_index: int32
        (b, stack_len) slot table; mask_bits: u8 (b, ceil(gh*gw/8)).
        Returns u8 (b, h, w, c) merged planes; with ``in_place`` each stream's
        corrupted plane (its last slot) becomes the merged plane and nothing
        is returned (no pass-through copy of the trusted pixels)."""
        # native: a handle the caller resolved once (serving loops), which
        # skips the per-call weight-change check
        nat = native if native is not None else self.model.native(frames.device)
        _, h, w, c = frames.shape
        b = frame_index.shape[0]
        if c != self.channels:
            raise ValueError("expected %d channels, got %d" % (self.channels, c))
        if in_place:
            return nat.recover_u8(frames, frame_index, mask_bits, None, b, h, w, self.precision)
        if out is None:
            out = torch.empty((b, h, w, c), dtype=torch.uint8, device=frames.device)
        return nat.recover_u8(frames, frame_index, mask_bits, out, b, h, w, self.precision)

    def recover_device16(self, frames: torch.Tensor, frame_index: torch.Tensor,
                         mask_bits: torch.Tensor, out: torch.Tensor | None = None,
                         in_place: bool = False, native=None) -> torch.Tensor | None:
        """``recover_device`` for 16-bit depth planes (``nvrec_recover_u16``):
        frames uint16 (n_slots, h, w) of a channels == 1 model, normalised as
        u16 / 65535 and quantised as ``clip(out * 65535 + 0.5, 0, 65535)``."""
        nat = native if native is not None else self.model.native(frames.device)
        if self.channels != 1:
            raise ValueError("16-bit planes need a depth (channels == 1) model")
        if frames.dtype != torch.uint16 or frames.dim() != 3:
            raise ValueError("frames must be uint16 (n_slots, h, w)")
        _, h, w = frames.shape
        b = frame_index.shape[0]
        if in_place:
            return nat.recover_u16(frames, frame_index, mask_bits, None, b, h, w, self.precision)
        if out is None:
            out = torch.empty((b, h, w), dtype=torch.uint16, device=frames.device)
        return nat.recover_u16(frames, frame_index, mask_bits, out, b, h, w, self.precision)

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


def cyclic_slot_tables(k: int, nbuf: int, n: int, F: int, device) -> torch.Tensor:
    """Slot tables of the cyclic slot-major ring (S = k + nbuf slots of n
    streams): phase p = step % S reads references p .. p+k-1 (mod S, oldest
    first, front-padded as ``stack_slots`` does) and the corrupted plane in
    slot p+k.  Returns int32 (S, n, F) flat indices slot * n + stream."""
    S = k + nbuf
    slots = stack_slots(k, k, F)
    tab = np.empty((S, n, F), np.int32)
    for p in range(S):
        ring = [(p + j) % S for j in range(k)] + [(p + k) % S]
        for s in range(n):
            tab[p, s] = [ring[x] * n + s for x in slots]
    return torch.from_numpy(tab).to(device)


def grid_shape(h: int, w: int) -> tuple[int, int]:
    return h // MASK_BLOCK, w // MASK_BLOCK


class RecoveryPipeline:
    """Pipelined multi-stream serving loop for one modality.

    A server hosting ``n`` conference streams of one resolution receives, per
    frame time, each stream's decoded corrupted plane and its P-frame shard
    state.  ``submit`` stages them (pinned host memory), then enqueues

      copy stream     H2D of the planes + loss-mask jobs into buffer i
      compute stream  nvrec_loss_mask -> nvrec_recover_u8 in place: the
                      recovered patches are written into the corrupted plane's
                      own slot, which then becomes the newest reference
                      (reference receiver.py:268-269) -- no pass-through copy,
                      no ring copies
      copy stream     D2H of the recovered planes

    with buffer i = step % nbuf, so the transfers of neighbouring steps
    overlap the compute.  Device memory is slot-major, ``frames[slot][stream]``
    with S = k + nbuf slots used cyclically (all streams advance together):
    step t reads the reference ring t .. t+k-1 (mod S, oldest first) and
    stages its corrupted plane in slot t+k, which joins the ring; slot t
    leaves it and is next written at step t+nbuf, after step t's compute.
    ``result(handle)`` waits for that step's D2H and returns the pinned host
    array (n, h, w, c); it stays valid for ``nbuf`` more submits."""

    def __init__(self, engine: RecoveryEngine, n: int, h: int, w: int,
                 shard_len: int, max_header: int, max_shards: int, init_refs: torch.Tensor,
                 nbuf: int = 3, graphs: bool = True, h2d_streams: int = 4):
        from .lossmask import LossMaskBatch
        self.engine = engine
        self.n, self.h, self.w = n, h, w
        self.c = engine.channels
        cfg = engine.model.config
        self.k, self.F = cfg.k, cfg.stack_len
        self.nbuf = nbuf
        dev = init_refs.device
        self.device = dev
        self.S = self.k + nbuf
        self.frames = torch.empty((self.S, n, h, w, self.c), dtype=torch.uint8, device=dev)
        self.frames[:self.k].copy_(init_refs.transpose(0, 1))      # (n, k, ...) -> slot-major
        self.flat = self.frames.view(self.S * n, h, w, self.c)
        self.nblk = (h // 16) * (w // 16)
        self.lm = [LossMaskBatch(n, max_header, max_shards, self.nblk, 1, dev)
                   for _ in range(nbuf)]
        self.host_in = [torch.empty((n, h, w, self.c), dtype=torch.uint8).pin_memory()
                        for _ in range(nbuf)]
        self.host_out = [torch.empty((n, h, w, self.c), dtype=torch.uint8).pin_memory()
                         for _ in range(nbuf)]
        self.tables = cyclic_slot_tables(self.k, nbuf, n, self.F, dev)
        # per buffer set: the step's slot table, copied in with its inputs, so
        # one CUDA graph per buffer set serves every ring phase
        self.tab_cur = torch.empty((nbuf, n, self.F), dtype=torch.int32, device=dev)
        # a private weight snapshot for the pipeline's lifetime: its CUDA
        # graphs hold the packed weight pointers (re-create the pipeline to
        # serve new weights)
        self.nat = engine.model.native_snapshot(dev)
        self.s_h2d = torch.cuda.Stream(dev)
        # one DMA stream reaches ~40 GB/s host->device; four in parallel ~51
        self.s_parts = [torch.cuda.Stream(dev) for _ in range(max(1, min(h2d_streams, n)))]
        self.s_cmp = torch.cuda.Stream(dev)
        self.s_d2h = torch.cuda.Stream(dev)
        self.ev_h2d = [torch.cuda.Event() for _ in range(nbuf)]
        self.ev_cmp = [torch.cuda.Event() for _ in range(nbuf)]
        self.ev_d2h = [torch.cuda.Event() for _ in range(nbuf)]
        self.step = 0
        self.shard_len = shard_len
        self.use_graphs = graphs
        self._graphs = {}

    def h2d_bytes(self) -> int:
        return int(self.host_in[0].numel() + self.lm[0].h2d_bytes)

    def d2h_bytes(self) -> int:
        return int(self.host_out[0].numel())

    def _compute(self, i: int, stream) -> None:
        lib = self.lm[i].lib
        with torch.cuda.stream(stream):
            _native.check(lib.nvrec_loss_mask(ctypes.c_void_p(self.lm[i].dev_in.data_ptr()),
                                              self.lm[i].n,
                                              ctypes.c_void_p(int(stream.cuda_stream))))
            self.engine.recover_device(self.flat, self.tab_cur[i], self.lm[i].wire,
                                       in_place=True, native=self.nat)

    def _run(self, i: int) -> None:
        if not self.use_graphs:
            self._compute(i, self.s_cmp)
            return
        g = self._graphs.get(i)
        if g is None:
            # warm the launch paths (attributes, workspace) outside capture
            with torch.cuda.stream(self.s_cmp):
                self._compute(i, self.s_cmp)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.s_cmp):
                self._compute(i, self.s_cmp)
            self._graphs[i] = g
            # the warm-up consumed this step's inputs and wrote the output
            # slot once; replaying recomputes the same values, so replay only
            # where the warm-up result is not already final
            return
        with torch.cuda.stream(self.s_cmp):
            g.replay()

    def submit(self, planes: np.ndarray | None, frames) -> int:
        """planes: (n, h, w, c) u8 host array (or None if already written into
        ``host_in[step % nbuf]``); frames: n ``PFrameShards``.  Returns a handle."""
        i = self.step % self.nbuf
        if self.step >= self.nbuf:
            self.ev_h2d[i].synchronize()          # staging buffers of step - nbuf are free
            self.ev_d2h[i].synchronize()          # host_out[i] consumed by the caller
        if planes is not None:
            self.host_in[i].numpy()[...] = planes
        self.lm[i].stage(frames)
        ph = self.step % self.S
        st = (self.step + self.k) % self.S             # this step's corrupted-plane slot
        # H2D: planes into the corrupted-plane slot, loss-mask jobs
        if self.step >= self.nbuf:
            self.s_h2d.wait_event(self.ev_cmp[i])  # step - nbuf read slot st (its oldest ref)
        start = self.s_h2d.record_event()
        per = -(-self.n // len(self.s_parts))
        for p, sp in enumerate(self.s_parts):
            lo, hi = p * per, min(self.n, (p + 1) * per)
            if lo >= hi:
                continue
            sp.wait_event(start)
            with torch.cuda.stream(sp):
                self.frames[st, lo:hi].copy_(self.host_in[i][lo:hi], non_blocking=True)
            self.s_h2d.wait_stream(sp)
        with torch.cuda.stream(self.s_h2d):
            self.lm[i].dev_in.copy_(self.lm[i].host, non_blocking=True)
            self.tab_cur[i].copy_(self.tables[ph], non_blocking=True)
            self.ev_h2d[i].record(self.s_h2d)
        # compute: the recovered patches land in slot st itself
        self.s_cmp.wait_event(self.ev_h2d[i])
        self._run(i)
        self.ev_cmp[i].record(self.s_cmp)
        # D2H of the recovered planes (now the newest references)
        self.s_d2h.wait_event(self.ev_cmp[i])
        with torch.cuda.stream(self.s_d2h):
            self.host_out[i].copy_(self.frames[st], non_blocking=True)
            self.ev_d2h[i].record(self.s_d2h)
        self.step += 1
        return i

    def result(self, handle: int) -> np.ndarray:
        self.ev_d2h[handle].synchronize()
        return self.host_out[handle].numpy()

    def status(self, handle: int) -> np.ndarray:
        """Per-stream loss-mask status of a step (0 = ok; else the header was
        undecodable -- LOST_FRAME in the reference receiver, receiver.py:
        244-248 -- and the kernel cleared that stream's wire bits, so its
        plane was returned exactly as submitted)."""
        self.ev_d2h[handle].synchronize()
        return self.lm[handle].status[:self.n, 0].cpu().numpy()


def recover_depth16(model, plane: np.ndarray, grid: np.ndarray, refs: list,
                    precision: str | None = None) -> np.ndarray:
    """16-bit depth extension of ``_recover`` (SPEC.md:74 calls 16-bit depth
    an extension point; the reference codec and wire format are u8-only).

    Planes are u16 (h, w), normalised as ``u16 / 65535`` (the 16-bit analogue
    of server.py:189), the output quantised with ``clip(out * 65535 + 0.5, 0,
    65535)`` and merged through the block mask -- all inside one
    ``nvrec_recover_u16`` call (the u16 planes go to the device as they are;
    the embedding reads each pixel as its two bytes).  Use the precise path
    (the model's precision by default): it keeps the error below 1/65535 of
    full scale (the north_star's <= 1 mm at 1 mm per depth unit)."""
    plane = np.asarray(plane)
    if not refs or not np.asarray(grid).any():
        return np.ascontiguousarray(plane)
    cfg = model.config
    dev = _native.require_cuda()
    refs = list(refs)[-cfg.k:]
    host = np.stack([np.asarray(r, dtype=np.uint16) for r in refs] + [plane.astype(np.uint16)])
    slots = stack_slots(len(refs), cfg.k, cfg.stack_len)
    frames = torch.from_numpy(host).to(dev, non_blocking=True)
    index = torch.tensor([slots], dtype=torch.int32).to(dev, non_blocking=True)
    bits = torch.from_numpy(pack_grid(grid)[None]).to(dev, non_blocking=True)
    eng = RecoveryEngine(model, precision or getattr(model, "precision", "precise"))
    return eng.recover_device16(frames, index, bits)[0].cpu().numpy()
