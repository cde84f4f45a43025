"""Oracle: restatement of the P-frame loss-mask construction.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The reference builds the corruption mask in three places; each function
below restates one of them with numpy:

* ``zero_fill_ranges``   -- ``Receiver._finalize_p`` (receiver.py:224-237):
  every missing body shard i in [1, n_data) zero-fills payload bytes
  ``[(i-1)*L, min(i*L, body_len))``.
* ``parse_header``       -- ``codec.parse_header`` (codec.py:180-201) and
  ``_Header.block_ranges`` (codec.py:172-177).
* ``corrupted_blocks``   -- ``codec._corrupted_blocks`` (codec.py:250-257).
* ``decode_mask``        -- the mask half of ``codec.decode``
  (codec.py:271-281,318-320) including the short-payload tail rule.
* ``wire_bits``          -- ``np.packbits`` of the grid (recovery.py:221).
"""

from __future__ import annotations

import struct

import numpy as np

HDR_FMT = "<BBHHBBIH"          # codec.py:26
HDR_FIXED = struct.calcsize(HDR_FMT)   # 14 bytes


class UndecodableError(ValueError):
    """codec.py:30-31."""


def parse_header(data: bytes) -> dict:
    """codec.py:180-201."""
    if len(data) < HDR_FIXED:
        raise UndecodableError("header truncated")
    kind, ch, w, h, block, quant, payload_len, n_present = \
        struct.unpack_from(HDR_FMT, data)
    if block == 0 or w % block or h % block:
        raise UndecodableError("inconsistent geometry in header")
    n_blocks = (w // block) * (h // block)
    bitmap_len = (n_blocks + 7) // 8
    hdr_len = HDR_FIXED + bitmap_len + 4 * n_present
    if len(data) < hdr_len:
        raise UndecodableError("header truncated")
    present = np.unpackbits(np.frombuffer(data, np.uint8, bitmap_len, HDR_FIXED),
                            count=n_blocks).astype(bool)
    if int(present.sum()) != n_present:
        raise UndecodableError("bitmap disagrees with present count")
    offsets = np.frombuffer(data, "<u4", n_present,
                            HDR_FIXED + bitmap_len).astype(np.int64)
    if kind not in (0, 1):                 # _Header(FrameKind(kind), ...) (codec.py:200)
        raise ValueError("%d is not a valid FrameKind" % kind)
    return dict(kind=kind, channels=ch, width=w, height=h, block=block,
                quant=quant, payload_len=payload_len, present=present,
                offsets=offsets, header_len=hdr_len)


def block_ranges(hdr: dict) -> np.ndarray:
    """codec.py:172-177: (n_present, 2) [start, end) payload byte ranges."""
    off = hdr["offsets"]
    if len(off) == 0:
        return np.zeros((0, 2), np.int64)
    ends = np.concatenate((off[1:], [hdr["payload_len"]]))
    return np.stack((off, ends), axis=1)


def corrupted_blocks(ranges: np.ndarray, zero_fill) -> np.ndarray:
    """codec.py:250-257: flag ranges intersecting any non-empty zero range."""
    flagged = np.zeros(len(ranges), bool)
    for z0, z1 in zero_fill:
        if z1 <= z0:
            continue
        flagged |= (ranges[:, 0] < z1) & (ranges[:, 1] > z0)
    return flagged


def decode_mask(header: bytes, received_payload_len: int, zero_fill) -> np.ndarray:
    """Mask half of ``codec.decode`` (codec.py:267-281,318-320).

    ``received_payload_len`` is ``len(enc.payload)``; when it is shorter than
    the header's ``payload_len`` the missing tail counts as zero-filled
    (codec.py:274-278).  Returns the (h/block, w/block) bool grid."""
    hdr = parse_header(header)
    zf = list(zero_fill)
    if received_payload_len < hdr["payload_len"]:
        zf.append((received_payload_len, hdr["payload_len"]))
    flagged = corrupted_blocks(block_ranges(hdr), zf)
    grid = np.zeros(len(hdr["present"]), bool)
    grid[np.flatnonzero(hdr["present"])[flagged]] = True
    b = hdr["block"]
    return grid.reshape(hdr["height"] // b, hdr["width"] // b)


def zero_fill_ranges(n_data: int, received, shard_len: int, body_len: int):
    """receiver.py:224-237 (ranges only; the body bytes are not needed)."""
    out = []
    for i in range(1, n_data):
        lo = (i - 1) * shard_len
        hi = min(lo + shard_len, body_len)
        if i not in received:
            out.append((lo, hi))
    return out


def mask_from_shards(header: bytes, n_data: int, received, shard_len: int,
                     encoded_len: int) -> np.ndarray:
    """Receiver -> codec path for one P-frame whose header arrived.

    body_len = encoded_len - len(header) (receiver.py:225); the assembled
    body has exactly body_len bytes (received shards are full slices,
    packet.py:121-127), so the tail rule does not fire on this path."""
    body_len = encoded_len - len(header)
    zf = zero_fill_ranges(n_data, received, shard_len, body_len)
    return decode_mask(header, body_len, zf)


def wire_bits(grid: np.ndarray) -> bytes:
    """recovery.py:221."""
    return np.packbits(np.asarray(grid, bool).reshape(-1)).tobytes()
