"""Synthetic workload generators for the benchmark and tests (no reference
code needed on the GPU box).  WORKLOAD INFRASTRUCTURE, not product code:
nothing in ``paper_2604_27441_b200/`` imports it; ``bench.py`` and
``tests/`` use it to synthesise the sender side (encoded P-frames, shard
plans, channel loss) that the recovery path consumes.

* ``p_frame_header`` -- a codec P-frame header with the reference layout
  (codec.py:26,146-153: ``<BBHHBBIH`` + MSB-first present bitmap + u32
  per-block payload offsets) and payload sizes in whole 3-byte RLE records
  (codec.py:25), as produced for partially changed frames.
* ``GilbertElliott`` -- the two-state loss process of
  rgbdstream/channel.py:59-121 (same draw order per packet).
* ``p_frame_shards`` -- shard plan of a P-frame (fec.py:249-254,
  packet.py:121-127): shard 0 = header, ``1 + ceil(body/L)`` data shards.
"""

from __future__ import annotations

import math
import struct

import numpy as np

RLE_RECORD = 3


def p_frame_header(rng: np.random.Generator, width: int, height: int, channels: int,
                   present_ratio: float = 0.1, block: int = 16, quant: int = 4):
    """Return (header bytes, payload_len)."""
    gh, gw = height // block, width // block
    n = gh * gw
    present = rng.random(n) < present_ratio
    np_ = int(present.sum())
    # records per changed block: 1 .. block*block*channels, skewed small
    max_rec = block * block * channels
    recs = np.minimum(max_rec, 1 + rng.geometric(1.0 / (8 * channels), np_))
    sizes = recs * RLE_RECORD
    offsets = np.concatenate(([0], np.cumsum(sizes)[:-1])).astype("<u4")
    payload_len = int(sizes.sum())
    head = struct.pack("<BBHHBBIH", 1, channels, width, height, block, quant,
                       payload_len, np_)
    return head + np.packbits(present).tobytes() + offsets.tobytes(), payload_len


class GilbertElliott:
    """GEModel + _GEState (channel.py:59-78,106-121)."""

    def __init__(self, p_gb=0.0155, p_bg=0.5, loss_good=0.0, loss_bad=1.0, seed=0):
        self.p_gb, self.p_bg = p_gb, p_bg
        self.loss_good, self.loss_bad = loss_good, loss_bad
        self.rng = np.random.default_rng(seed)
        self.bad = False

    def drop(self) -> bool:
        if self.bad:
            if self.rng.random() < self.p_bg:
                self.bad = False
        elif self.rng.random() < self.p_gb:
            self.bad = True
        p = self.loss_bad if self.bad else self.loss_good
        return bool(self.rng.random() < p)


def n_data_shards(body_len: int, shard_len: int) -> int:
    """fec.py:250: shard 0 (header) + ceil(body/L) body shards."""
    return 1 + math.ceil(body_len / shard_len) if body_len > 0 else 1


def p_frame_shards(rng, width, height, channels, shard_len, loss, present_ratio=0.1):
    """One synthetic P-frame as the receiver sees it at its deadline:
    (header, n_data, received bool[n_data], encoded_len).  ``loss`` is a
    callable returning True to drop a body shard (header always kept)."""
    header, payload_len = p_frame_header(rng, width, height, channels, present_ratio)
    nd = n_data_shards(payload_len, shard_len)
    received = np.ones(nd, bool)
    for i in range(1, nd):
        received[i] = not loss()
    return header, nd, received, len(header) + payload_len


# ---------------------------------------------------------------------------
# Sender side of the codec + FEC, for building receiver workloads on the GPU
# box (where the reference is absent).  Vectorised restatements of
# rgbdstream codec.encode_i / encode_p (codec.py:212-247) with _blockify,
# _rle_encode, _zigzag and _pack_header (codec.py:85-157), and fec.rs_encode
# (fec.py:115-141).  tests/test_codec_oracle.py checks them byte-for-byte
# against fixtures made by the reference encoder.

KIND_I, KIND_P = 0, 1
_HDR = "<BBHHBBIH"


def _blockify(plane: np.ndarray, block: int) -> np.ndarray:
    if plane.ndim == 2:
        plane = plane[:, :, None]
    h, w, c = plane.shape
    a = plane.reshape(h // block, block, w // block, block, c).transpose(0, 2, 4, 1, 3)
    return a.reshape((h // block) * (w // block), block * block * c)


def _rle_encode(vals: np.ndarray, bs: int):
    n = len(vals)
    if n == 0:
        return b"", np.zeros(0, np.int64)
    change = np.flatnonzero(vals[1:] != vals[:-1]) + 1
    starts = np.union1d(np.concatenate(([0], change)), np.arange(0, n, bs))
    lengths = np.diff(np.concatenate((starts, [n])))
    nchunks = (lengths + 254) // 255
    total = int(nchunks.sum())
    run_vals = np.repeat(vals[starts], nchunks)
    run_lens = np.full(total, 255, np.int64)
    last = np.cumsum(nchunks) - 1
    run_lens[last] = lengths - (nchunks - 1) * 255
    rec = np.empty((total, 3), np.uint8)
    rec[:, 0] = run_lens
    rec[:, 1] = run_vals & 0xFF
    rec[:, 2] = run_vals >> 8
    per_block = np.bincount(np.repeat(starts // bs, nchunks), minlength=n // bs)
    offsets = np.concatenate(([0], np.cumsum(per_block[:-1]))) * 3
    return rec.tobytes(), offsets


def _header(kind, c, h, w, block, quant, payload_len, present, offsets) -> bytes:
    return (struct.pack(_HDR, kind, c, w, h, block, quant, payload_len, int(present.sum()))
            + np.packbits(present).tobytes() + np.asarray(offsets).astype("<u4").tobytes())


def encode_i(plane: np.ndarray, quant: int = 4, block: int = 16):
    """codec.py:212-222 -> (header, payload)."""
    h, w = plane.shape[:2]
    c = 1 if plane.ndim == 2 else plane.shape[2]
    q = (plane.astype(np.uint16) + quant // 2) // quant
    vals = _blockify(q, block).reshape(-1)
    bs = block * block * c
    payload, offsets = _rle_encode(vals, bs)
    present = np.ones(len(vals) // bs, bool)
    return _header(KIND_I, c, h, w, block, quant, len(payload), present, offsets), payload


def encode_p(plane: np.ndarray, reference: np.ndarray, quant: int = 4, block: int = 16):
    """codec.py:225-247 -> (header, payload)."""
    h, w = plane.shape[:2]
    c = 1 if plane.ndim == 2 else plane.shape[2]
    d = plane.astype(np.int32) - reference.astype(np.int32)
    qd = np.sign(d) * (np.abs(d) // quant)
    blocks = _blockify(qd.astype(np.int16), block)
    present = (blocks != 0).any(axis=1)
    v = blocks[present].reshape(-1).astype(np.int16)
    vals = ((v << 1) ^ (v >> 15)).astype(np.uint16)
    payload, offsets = _rle_encode(vals, block * block * c)
    return _header(KIND_P, c, h, w, block, quant, len(payload), present, offsets), payload


def _gf_tables():
    exp = np.zeros(512, np.uint8)
    log = np.zeros(256, np.int32)
    x = 1
    for i in range(255):
        exp[i], log[x] = x, i
        x <<= 1
        if x & 0x100:
            x ^= 0x11D
    exp[255:510] = exp[:255]
    mul = np.zeros((256, 256), np.uint8)
    a = np.arange(1, 256)
    mul[1:, 1:] = exp[(log[a][:, None] + log[a][None, :]) % 255]
    return mul


_GF_MUL = None


def _gf_inv(m: np.ndarray, mul) -> np.ndarray:
    n = m.shape[0]
    aug = np.concatenate((m.copy(), np.eye(n, dtype=np.uint8)), axis=1)
    inv_of = np.zeros(256, np.uint8)
    for a in range(1, 256):
        inv_of[a] = np.flatnonzero(mul[a] == 1)[0]
    for col in range(n):
        piv = col + int(np.argmax(aug[col:, col] != 0))
        if piv != col:
            aug[[col, piv]] = aug[[piv, col]]
        aug[col] = mul[inv_of[aug[col, col]], aug[col]]
        f = aug[:, col].copy()
        f[col] = 0
        aug ^= mul[f[:, None], aug[col][None, :]]
    return aug[:, n:]


def rs_parity(data: bytes, n: int, r: int, shard_len: int) -> list[bytes]:
    """fec.py:115-141: the r parity shards of ``data`` split into n shards."""
    global _GF_MUL
    if _GF_MUL is None:
        _GF_MUL = _gf_tables()
    mul = _GF_MUL
    padded = np.frombuffer(data.ljust(n * shard_len, b"\x00"), np.uint8).reshape(n, shard_len)
    if r == 0:
        return []
    points = np.arange(n + r, dtype=np.uint8)
    vand = np.zeros((n + r, n), np.uint8)
    vand[:, 0] = 1
    for j in range(1, n):
        vand[:, j] = mul[vand[:, j - 1], points]
    top_inv = _gf_inv(vand[:n], mul)
    gen = np.bitwise_xor.reduce(mul[vand[n:, :, None], top_inv[None, :, :]], axis=1)
    parity = np.zeros((r, shard_len), np.uint8)
    for i in range(r):
        for j in range(n):
            parity[i] ^= mul[gen[i, j]][padded[j]]
    return [parity[i].tobytes() for i in range(r)]


def i_frame_plan(encoded_len: int, payload_len: int, ratio: float = 0.5):
    """fec.py:233-247 (REVO mode): (n, r, shard_len) of an I-frame."""
    shard_len = payload_len
    while True:
        n = math.ceil(encoded_len / shard_len)
        r = math.ceil(ratio * n)
        if n + r <= 255:
            return n, r, shard_len
        shard_len *= 2


def talking_clip(n_frames: int, width: int, height: int, channels: int, seed: int = 0,
                 motion_fraction: float = 0.07, cell: int = 8):
    """Synthetic conference content: a static coarse-textured background with
    a re-textured, slowly moving foreground patch covering ~motion_fraction
    of the frame (the workload shape of rgbdstream's talking-motion clips:
    P-frames touch a few percent of the blocks).  Returns u8 planes
    (h, w[, c])."""
    rng = np.random.default_rng(seed)

    def coarse(h, w, c, lo, hi):
        g = rng.integers(lo, hi, (h // cell + 1, w // cell + 1, c), dtype=np.uint8)
        return np.repeat(np.repeat(g, cell, 0), cell, 1)[:h, :w]

    lo, hi = (0, 256) if channels == 3 else (150, 230)
    bg = coarse(height, width, channels, lo, hi)
    pw = max(cell, int(width * math.sqrt(motion_fraction)))
    ph = max(cell, int(height * math.sqrt(motion_fraction)))
    cy, cx = (height - ph) // 2, (width - pw) // 2
    out = []
    for i in range(n_frames):
        y0 = int(np.clip(cy + int(3 * math.sin(i / 3.0)), 0, height - ph))
        x0 = int(np.clip(cx + int(4 * math.cos(i / 4.0)), 0, width - pw))
        f = bg.copy()
        f[y0:y0 + ph, x0:x0 + pw] = coarse(ph, pw, channels, lo // 2, hi // 2 + 40)
        out.append(f if channels == 3 else f[:, :, 0])
    return out


def receiver_body(payload: bytes, shard_len: int, received) -> bytes:
    """Receiver._finalize_p body assembly (receiver.py:228-237): received body
    shards verbatim, zero chunks for the missing ones."""
    out = bytearray(payload)
    for i in range(1, len(received)):
        if not received[i]:
            lo = (i - 1) * shard_len
            out[lo:lo + shard_len] = b"\0" * len(out[lo:lo + shard_len])
    return bytes(out)
