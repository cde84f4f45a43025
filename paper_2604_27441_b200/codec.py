"""Frame decode and I-frame FEC on the GPU.

Drop-in for the two reference steps that produce the recovery path's input:

* ``decode`` / ``decode_bytes`` -- ``rgbdstream.codec.decode`` /
  ``decode_bytes`` (codec.py:260-340): zero-fill P-frame (or I-frame) decode
  returning the corrupted plane and its ``CorruptionMask``, same errors
  (``UndecodableError`` messages, ``ValueError`` for a P-frame without a
  reference or an invalid frame kind).
* ``rs_reconstruct`` -- ``rgbdstream.fec.rs_reconstruct`` (fec.py:144-163)
  over a duck-typed ``ShardSet``; ``UnrecoverableError`` when fewer than n
  shards survive.

Both are thin hosts around ``nvrec_decode`` / ``nvrec_rs_plan`` +
``nvrec_rs_reconstruct`` (k_decode.cu, k_rs.cu).  ``DecodeBatch`` is the
serving form: fixed-capacity pinned staging, one H2D copy and four kernel
launches for a batch of frames, outputs (planes, grids, wire bitsets) left on
the device for ``nvrec_recover_u8``.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .lossmask import HDR_FIXED, UndecodableError

KIND_I, KIND_P = 0, 1

_STATUS = {1: "header truncated", 2: "inconsistent geometry in header",
           3: "header truncated", 4: "bitmap disagrees with present count",
           6: "payload range is not whole RLE records",
           7: "payload sample count disagrees with header"}


class UnrecoverableError(Exception):
    """Fewer than n shards survive (fec.py:91-92)."""


class CorruptionMask:
    """Per-block grid, True = payload fell in a zeroed range (codec.py:64-82)."""

    def __init__(self, grid: np.ndarray):
        self.grid = np.asarray(grid, dtype=bool)
        self.grid.setflags(write=False)

    @property
    def any(self) -> bool:
        return bool(self.grid.any())

    def to_pixels(self, block: int, channels: int = 1) -> np.ndarray:
        m = np.repeat(np.repeat(self.grid, block, axis=0), block, axis=1)
        if channels > 1:
            m = np.repeat(m[:, :, None], channels, axis=2)
        return m


def raise_status(code: int, header: bytes = b"") -> None:
    if code == 0:
        return
    if code in _STATUS:
        raise UndecodableError(_STATUS[code])
    if code == 8:
        raise ValueError("P-frame decode requires a reference plane")
    if code == 10:
        raise ValueError("%d is not a valid FrameKind" % (header[0] if header else -1))
    raise ValueError("decode capacity exceeded (status %d)" % code)


def header_geometry(header: bytes):
    """(kind, channels, h, w, block) of a codec header, or None if malformed."""
    if len(header) < HDR_FIXED:
        return None
    kind, c, w, h, block, _, _, _ = struct.unpack_from("<BBHHBBIH", header)
    if block == 0 or w % block or h % block:
        return None
    return kind, c, h, w, block


@dataclass
class DecodeItem:
    """One frame of a ``DecodeBatch``.

    ``payload`` is the assembled payload (``len(enc.payload)`` bytes; the
    receiver's body with zero chunks for missing shards).  Zero-filled
    ranges come either explicitly (``zero_fill_ranges``, codec level) or in
    receiver form (``n_data`` / ``received`` / ``shard_len`` / ``body_len``,
    receiver.py:224-237).  ``reference`` / ``out`` are device u8 planes
    (h, w, c); ``out`` may alias ``reference``."""
    header: bytes
    payload: object
    out: torch.Tensor
    reference: torch.Tensor | None = None
    zero_fill_ranges: tuple = ()
    n_data: int = 1
    received: object = None
    shard_len: int = 1
    body_len: int = 0


class DecodeBatch:
    """Fixed-capacity batch runner for ``nvrec_decode``."""

    def __init__(self, max_jobs: int, max_header: int, max_payload: int, max_blocks: int,
                 max_shards: int = 256, max_ranges: int = 8, device=None):
        self.lib = _native.load_library()
        self.device = _native.require_cuda(device)
        self.max_jobs, self.max_header, self.max_payload = max_jobs, max_header, max_payload
        self.max_blocks, self.max_shards, self.max_ranges = max_blocks, max_shards, max_ranges
        js = ctypes.sizeof(_native.DecodeJob)
        al = lambda n: (n + 255) // 256 * 256
        # [jobs | headers | shard flags | ranges | payloads packed back to
        # back]: the used prefix goes to the device in ONE copy
        self.o_hdr = al(js * max_jobs)
        self.o_recv = self.o_hdr + al(max_jobs * max_header)
        self.o_rng = self.o_recv + al(max_jobs * max_shards)
        self.o_pay = self.o_rng + al(max_jobs * max_ranges * 16)
        self.in_bytes = self.o_pay + al(max_jobs * (max_payload + 16))
        self.used = self.o_pay
        self.host = torch.empty(self.in_bytes, dtype=torch.uint8, pin_memory=True)
        self.dev_in = torch.empty(self.in_bytes, dtype=torch.uint8, device=self.device)
        self.grid = torch.zeros((max_jobs, max_blocks), dtype=torch.uint8, device=self.device)
        self.wire_stride = (max_blocks + 7) // 8
        self.wire = torch.zeros((max_jobs, self.wire_stride), dtype=torch.uint8,
                                device=self.device)
        self.status = torch.zeros((max_jobs, 4), dtype=torch.int32, device=self.device)
        self.scratch = torch.zeros((max_jobs, 2 * max_blocks + 4), dtype=torch.int32,
                                   device=self.device)
        self._jobs = (_native.DecodeJob * max_jobs)()
        self.n = 0
        self.h2d_bytes = 0
        self.headers = []

    def stage(self, items: list[DecodeItem]) -> None:
        if len(items) > self.max_jobs:
            raise ValueError("batch of %d frames exceeds capacity %d" % (len(items), self.max_jobs))
        hb = self.host.numpy()
        base = self.dev_in.data_ptr()
        end_pay = self.o_pay
        self.headers = []
        for j, it in enumerate(items):
            hdr = bytes(it.header)
            pay = np.frombuffer(bytes(it.payload), np.uint8) \
                if not isinstance(it.payload, np.ndarray) else it.payload.reshape(-1)
            if len(hdr) > self.max_header or pay.size > self.max_payload:
                raise ValueError("frame %d exceeds header/payload capacity" % j)
            if len(it.zero_fill_ranges) > self.max_ranges or it.n_data > self.max_shards:
                raise ValueError("frame %d exceeds range/shard capacity" % j)
            ho = self.o_hdr + j * self.max_header
            hb[ho:ho + len(hdr)] = np.frombuffer(hdr, np.uint8)
            po = end_pay
            hb[po:po + pay.size] = pay
            end_pay = po + (pay.size + 15) // 16 * 16
            ro = self.o_recv + j * self.max_shards
            if it.received is not None:
                hb[ro:ro + it.n_data] = np.asarray(it.received, np.uint8)[:it.n_data]
            else:
                hb[ro:ro + it.n_data] = 1
            go = self.o_rng + j * self.max_ranges * 16
            if it.zero_fill_ranges:
                rr = np.asarray(it.zero_fill_ranges, np.int64).reshape(-1)
                hb[go:go + rr.nbytes] = rr.view(np.uint8)
            job = self._jobs[j]
            mk = job.mask
            mk.header, mk.header_len = base + ho, len(hdr)
            mk.n_data, mk.received = it.n_data, base + ro
            mk.shard_len, mk.body_len = max(1, it.shard_len), it.body_len
            mk.payload_received = int(pay.size)
            mk.extra_ranges = base + go if it.zero_fill_ranges else None
            mk.n_extra = len(it.zero_fill_ranges)
            mk.grid = self.grid[j].data_ptr()
            mk.wire_bits = self.wire[j].data_ptr()
            mk.status = self.status[j].data_ptr()
            mk.grid_capacity = self.max_blocks
            job.payload = base + po
            if it.reference is not None and it.reference.numel() < it.out.numel():
                # the error policy copies plane_capacity bytes of the reference
                raise ValueError("frame %d: reference smaller than the output plane" % j)
            job.reference = it.reference.data_ptr() if it.reference is not None else None
            job.plane = it.out.data_ptr()
            job.plane_capacity = it.out.numel()
            job.scratch = self.scratch[j].data_ptr()
            self.headers.append(hdr)
        raw = bytes(self._jobs)[:ctypes.sizeof(_native.DecodeJob) * len(items)]
        hb[:len(raw)] = np.frombuffer(raw, np.uint8)
        self.n = len(items)
        self.used = end_pay
        self.h2d_bytes = self.used

    def launch(self, stream=None, copy: bool = True) -> None:
        s = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            if copy:
                self.dev_in[:self.used].copy_(self.host[:self.used], non_blocking=True)
            _native.check(self.lib.nvrec_decode(ctypes.c_void_p(self.dev_in.data_ptr()),
                                                self.n, self.max_blocks,
                                                ctypes.c_void_p(int(s.cuda_stream))))

    def check(self) -> list[tuple[int, int]]:
        """Synchronise; raise the first frame's error; return (gh, gw) per frame."""
        st = self.status[:self.n].cpu().numpy()
        out = []
        for j in range(self.n):
            raise_status(int(st[j, 0]), self.headers[j])
            out.append((int(st[j, 2]), int(st[j, 3])))
        return out

    def grids(self) -> list[np.ndarray]:
        shapes = self.check()
        g = self.grid[:self.n].cpu().numpy()
        return [g[j, :gh * gw].astype(bool).reshape(gh, gw) for j, (gh, gw) in enumerate(shapes)]


def decode(enc, reference=None, zero_fill_ranges=(), *, device=None):
    """``codec.decode(enc, reference, zero_fill_ranges)`` on the GPU.

    ``enc`` has ``.header`` and ``.payload`` (an ``EncodedFrame``) or is a
    (header, payload) pair.  ``reference`` is a host u8 plane (h, w[, c]) or
    a device tensor.  Returns (host plane, CorruptionMask)."""
    header, payload = (enc.header, enc.payload) if hasattr(enc, "header") else enc
    header, payload = bytes(header), bytes(payload)
    geo = header_geometry(header)
    dev = _native.require_cuda(device)
    if geo is None:
        raise_status(1 if len(header) < HDR_FIXED else 2)
    kind, c, h, w, block = geo
    ref_t = None
    if reference is not None:
        ref_t = reference if isinstance(reference, torch.Tensor) else \
            torch.from_numpy(np.ascontiguousarray(reference))
        if ref_t.numel() != h * w * c:
            raise ValueError("reference shape %r does not match the %dx%dx%d frame"
                             % (tuple(ref_t.shape), h, w, c))
        ref_t = ref_t.to(dev).reshape(h, w, c).contiguous()
    out = torch.empty((h, w, c), dtype=torch.uint8, device=dev)
    nblk = (h // block) * (w // block)
    zr = tuple(tuple(int(v) for v in r) for r in zero_fill_ranges)
    batch = DecodeBatch(1, max(len(header), HDR_FIXED), max(len(payload), 1), max(nblk, 1),
                        max_shards=1, max_ranges=max(1, len(zr)), device=dev)
    batch.stage([DecodeItem(header, payload, out, ref_t, zr)])
    batch.launch()
    grid = batch.grids()[0]
    plane = out.cpu().numpy()
    return (plane[:, :, 0] if c == 1 else plane), CorruptionMask(grid)


def decode_bytes(data: bytes, reference=None, zero_fill_ranges=(), *, device=None, **_):
    """``codec.decode_bytes`` (codec.py:324-340): ranges relative to the
    whole encoded frame; a range overlapping the header is undecodable."""
    data = bytes(data)
    geo = header_geometry(data)
    if geo is None:
        raise_status(1 if len(data) < HDR_FIXED else 2)
    n_present = struct.unpack_from("<H", data, 12)[0]
    kind, c, h, w, block = geo
    hl = HDR_FIXED + ((h // block) * (w // block) + 7) // 8 + 4 * n_present
    if len(data) < hl:
        raise UndecodableError("header truncated")
    pr = []
    for z0, z1 in zero_fill_ranges:
        if z0 < hl and z1 > 0 and z1 > z0:
            raise UndecodableError("zero-filled range overlaps codec header")
        pr.append((z0 - hl, z1 - hl))
    return decode((data[:hl], data[hl:]), reference, pr, device=device)


# ---- Reed-Solomon ------------------------------------------------------------------

def rs_plan(n: int, r: int, present):
    """Host decode plan (nvrec_rs_plan): (coef (m, n) u8, sources, missing)."""
    lib = _native.load_library()
    coef = np.zeros(max(1, r * n), np.uint8)
    src = np.zeros(n, np.int32)
    miss = np.zeros(max(1, r), np.int32)
    m = ctypes.c_int32()
    pres = np.ascontiguousarray(np.asarray(present, np.uint8))
    rc = lib.nvrec_rs_plan(n, r, pres.ctypes.data, coef.ctypes.data, src.ctypes.data,
                           miss.ctypes.data, ctypes.byref(m))
    if rc != 0:
        msg = lib.nvrec_last_error().decode()
        if "required shards present" in msg:
            raise UnrecoverableError(msg)
        raise ValueError(msg)
    return coef[:m.value * n].reshape(m.value, n), src, miss[:m.value]


def rs_reconstruct_device(data: torch.Tensor, parity: torch.Tensor, n: int, r: int,
                          shard_len: int, present, stream=None) -> int:
    """Fill the missing data rows of device ``data`` (n x shard_len u8, the
    present data shards already in place) from device ``parity`` (r x
    shard_len).  Returns the number of rows rebuilt."""
    coef, src, miss = rs_plan(n, r, present)
    m = len(miss)
    if m == 0:
        return 0
    dev = data.device
    s = stream or torch.cuda.current_stream(dev)
    c_t = torch.from_numpy(coef.reshape(-1).copy()).to(dev, non_blocking=False)
    s_t = torch.from_numpy(src).to(dev)
    m_t = torch.from_numpy(miss.copy()).to(dev)
    job = _native.RsJob(data.data_ptr(), parity.data_ptr() if parity is not None else None,
                        c_t.data_ptr(), s_t.data_ptr(), m_t.data_ptr(), n, r, m, shard_len)
    j_t = torch.frombuffer(bytearray(bytes(job)), dtype=torch.uint8).to(dev)
    aligned = int(shard_len % 4 == 0 and data.data_ptr() % 4 == 0 and
                  (parity is None or parity.data_ptr() % 4 == 0))
    with torch.cuda.stream(s):
        _native.check(_native.load_library().nvrec_rs_reconstruct(
            ctypes.c_void_p(j_t.data_ptr()), 1, shard_len, m * n, aligned,
            ctypes.c_void_p(int(s.cuda_stream))))
    # keep the small device buffers alive until the kernel has run
    s.synchronize()
    return m


def rs_reconstruct(s, device=None) -> bytes:
    """``fec.rs_reconstruct(ShardSet)`` on the GPU (fec.py:144-163)."""
    n, r, L = s.n, s.r, s.shard_len
    present = [bool(p) for p in s.present]
    if sum(present) < n:
        raise UnrecoverableError("only %d of %d required shards present" % (sum(present), n))
    if all(present[:n]):
        return b"".join(s.shards[:n])[:s.data_len]
    dev = _native.require_cuda(device)
    host = np.zeros((n, L), np.uint8)
    for i in range(n):
        if present[i]:
            host[i] = np.frombuffer(s.shards[i], np.uint8)
    par = np.zeros((max(r, 1), L), np.uint8)
    for i in range(r):
        if present[n + i]:
            par[i] = np.frombuffer(s.shards[n + i], np.uint8)
    data = torch.from_numpy(host).to(dev)
    parity = torch.from_numpy(par).to(dev)
    rs_reconstruct_device(data, parity, n, r, L, present)
    return data.cpu().numpy().reshape(-1).tobytes()[:s.data_len]
