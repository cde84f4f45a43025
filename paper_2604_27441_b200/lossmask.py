"""Loss-mask construction on the GPU (``nvrec_loss_mask``).

Replaces, bit-exactly, the reference's P-frame corruption-mask path:

* ``Receiver._finalize_p`` zero-fill of missing body shards
  (rgbdstream/receiver.py:224-237),
* ``codec.parse_header`` / ``_Header.block_ranges`` / ``_corrupted_blocks``
  and the mask assembly of ``codec.decode`` (codec.py:159-201,250-281,318-320),
* the wire bitset ``np.packbits(grid)`` (recovery.py:221).

``LossMaskBatch`` keeps fixed-capacity pinned staging and device buffers so
a batch of frames costs one H2D copy and one kernel launch, and its
``wire_bits`` output feeds ``nvrec_recover_u8`` without leaving the device.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native

HDR_FIXED = 14
_ERRORS = {1: "header truncated", 2: "inconsistent geometry in header",
           3: "header truncated", 4: "bitmap disagrees with present count",
           5: "grid capacity exceeded"}


class UndecodableError(ValueError):
    """Header is truncated or inconsistent (rgbdstream codec.py:30-31)."""


@dataclass
class PFrameShards:
    """What the receiver holds for one P-frame when its deadline fires.

    ``header`` is shard 0's payload (the codec header); ``received`` marks
    which of the ``n_data`` data shards arrived (index 0 = header);
    ``encoded_len`` is the DESC packet's ``encoded_frame_len``."""
    header: bytes
    n_data: int
    received: object          # iterable of indices, or bool sequence of n_data
    shard_len: int
    encoded_len: int
    payload_received: int | None = None      # default: body_len (receiver path)
    extra_ranges: tuple = ()                 # explicit codec zero-fill ranges

    def received_flags(self) -> np.ndarray:
        r = self.received
        if isinstance(r, np.ndarray) and r.dtype == bool:
            flags = r.astype(np.uint8)
        elif isinstance(r, (list, tuple)) and len(r) == self.n_data and \
                all(isinstance(v, (bool, np.bool_)) for v in r):
            flags = np.asarray(r, np.uint8)
        else:
            flags = np.zeros(self.n_data, np.uint8)
            for i in r:
                if 0 <= i < self.n_data:
                    flags[i] = 1
        return flags


def grid_blocks(header: bytes) -> int:
    """Block count the header declares (0 if the fixed part is malformed)."""
    if len(header) < HDR_FIXED:
        return 0
    _, _, w, h, block, _, _, _ = struct.unpack_from("<BBHHBBIH", header)
    if block == 0 or w % block or h % block:
        return 0
    return (w // block) * (h // block)


class LossMaskBatch:
    """Fixed-capacity batch runner for ``nvrec_loss_mask``."""

    def __init__(self, max_jobs: int, max_header: int, max_shards: int,
                 max_blocks: int, max_extra: int = 4, device=None):
        self.lib = _native.load_library()
        self.device = _native.require_cuda(device)
        self.max_jobs, self.max_header = max_jobs, max_header
        self.max_shards, self.max_blocks, self.max_extra = max_shards, max_blocks, max_extra
        self.wire_stride = (max_blocks + 7) // 8
        js = ctypes.sizeof(_native.LossMaskJob)
        al = lambda n: (n + 255) // 256 * 256
        self.o_jobs = 0
        self.o_hdr = al(js * max_jobs)
        self.o_recv = self.o_hdr + al(max_jobs * max_header)
        self.o_rng = self.o_recv + al(max_jobs * max_shards)
        in_bytes = self.o_rng + al(max_jobs * max_extra * 16)
        self.host = torch.empty(in_bytes, dtype=torch.uint8, pin_memory=True)
        self.dev_in = torch.empty(in_bytes, dtype=torch.uint8, device=self.device)
        self.grid = torch.zeros((max_jobs, max_blocks), dtype=torch.uint8, device=self.device)
        self.wire = torch.zeros((max_jobs, self.wire_stride), dtype=torch.uint8,
                                device=self.device)
        self.status = torch.zeros((max_jobs, 4), dtype=torch.int32, device=self.device)
        self.n = 0
        self._jobs = (_native.LossMaskJob * max_jobs)()
        self.h2d_bytes = 0

    def stage(self, frames: list[PFrameShards]) -> None:
        """Fill the pinned staging buffer for ``frames``."""
        if len(frames) > self.max_jobs:
            raise ValueError("batch of %d frames exceeds capacity %d"
                             % (len(frames), self.max_jobs))
        hb = self.host.numpy()
        base = self.dev_in.data_ptr()
        used = self.o_hdr
        for j, fr in enumerate(frames):
            hdr = bytes(fr.header)
            if len(hdr) > self.max_header or fr.n_data > self.max_shards:
                raise ValueError("frame %d exceeds header/shard capacity" % j)
            if len(fr.extra_ranges) > self.max_extra:
                raise ValueError("too many explicit zero-fill ranges")
            ho = self.o_hdr + j * self.max_header
            hb[ho:ho + len(hdr)] = np.frombuffer(hdr, np.uint8)
            ro = self.o_recv + j * self.max_shards
            hb[ro:ro + fr.n_data] = fr.received_flags()
            go = self.o_rng + j * self.max_extra * 16
            if fr.extra_ranges:
                rr = np.asarray(fr.extra_ranges, np.int64).reshape(-1)
                hb[go:go + rr.nbytes] = rr.view(np.uint8)
            body_len = fr.encoded_len - len(hdr)
            job = self._jobs[j]
            job.header, job.header_len = base + ho, len(hdr)
            job.n_data, job.received = fr.n_data, base + ro
            job.shard_len, job.body_len = fr.shard_len, body_len
            job.payload_received = body_len if fr.payload_received is None \
                else fr.payload_received
            job.extra_ranges = base + go if fr.extra_ranges else None
            job.n_extra = len(fr.extra_ranges)
            job.grid = self.grid[j].data_ptr()
            job.wire_bits = self.wire[j].data_ptr()
            job.status = self.status[j].data_ptr()
            job.grid_capacity = self.max_blocks
            used = max(used, ho + len(hdr))
        raw = bytes(self._jobs)[:ctypes.sizeof(_native.LossMaskJob) * len(frames)]
        hb[:len(raw)] = np.frombuffer(raw, np.uint8)
        self.n = len(frames)
        self.h2d_bytes = self.o_rng + self.max_jobs * self.max_extra * 16

    def launch(self, stream=None) -> None:
        """H2D of the staged batch + one kernel launch on ``stream``."""
        s = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            self.dev_in.copy_(self.host, non_blocking=True)
            _native.check(self.lib.nvrec_loss_mask(
                ctypes.c_void_p(self.dev_in.data_ptr()), self.n,
                ctypes.c_void_p(int(s.cuda_stream))))

    def results(self) -> list[np.ndarray]:
        """Synchronise and return each frame's (gh, gw) bool grid; raises
        ``UndecodableError`` like ``codec.parse_header``."""
        st = self.status[:self.n].cpu().numpy()
        grids = self.grid[:self.n].cpu().numpy()
        out = []
        for j in range(self.n):
            if st[j, 0]:
                raise UndecodableError(_ERRORS.get(int(st[j, 0]), "undecodable"))
            gh, gw = int(st[j, 2]), int(st[j, 3])
            out.append(grids[j, :gh * gw].astype(bool).reshape(gh, gw))
        return out


def loss_masks(frames: list[PFrameShards], device=None) -> list[np.ndarray]:
    """Convenience one-shot: corruption grids of a batch of P-frames."""
    if not frames:
        return []
    batch = LossMaskBatch(len(frames), max(len(f.header) for f in frames) + 16,
                          max(f.n_data for f in frames) + 1,
                          max(max(grid_blocks(f.header) for f in frames), 1),
                          max(4, max(len(f.extra_ranges) for f in frames)), device)
    batch.stage(frames)
    batch.launch()
    return batch.results()


def decode_mask(header: bytes, payload_received: int, zero_fill_ranges=(),
                device=None) -> np.ndarray:
    """GPU twin of the mask half of ``codec.decode(enc, ref, zero_fill)``:
    explicit zero-fill ranges, tail rule for a short payload."""
    fr = PFrameShards(header=header, n_data=1, received=[True], shard_len=1,
                      encoded_len=len(header) + payload_received,
                      payload_received=payload_received,
                      extra_ranges=tuple(tuple(r) for r in zero_fill_ranges))
    return loss_masks([fr], device)[0]
