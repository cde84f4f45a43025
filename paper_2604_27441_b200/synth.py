"""Synthetic workload generators for the benchmark and tests (no reference
code needed on the GPU box).

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
