"""GPU loss-mask kernel: bit-exact against the reference receiver+codec
(golden trials from tests/golden/make_golden.py) and the oracle on
synthetic and malformed headers."""

import os
import struct

import numpy as np
import pytest

from helpers import GOLDEN_DIR
from oracle import lossmask as om
from test_oracle_golden import LMASK, lossmask_trials

pytestmark = pytest.mark.gpu


def _lm():
    from paper_2604_27441_b200 import lossmask
    return lossmask


def test_kernel_matches_reference_receiver_golden():
    lm = _lm()
    trials = list(lossmask_trials())
    frames = [lm.PFrameShards(header=t["header"], n_data=t["n_data"],
                              received=t["received"].astype(bool),
                              shard_len=t["shard_len"], encoded_len=t["encoded_len"])
              for t in trials]
    grids = lm.loss_masks(frames)
    for t, g in zip(trials, grids):
        assert g.shape == (t["gh"], t["gw"])
        assert np.array_equal(g.reshape(-1), t["grid"])


def test_wire_bits_are_packbits():
    lm = _lm()
    trials = list(lossmask_trials())[:64]
    frames = [lm.PFrameShards(t["header"], t["n_data"], t["received"].astype(bool),
                              t["shard_len"], t["encoded_len"]) for t in trials]
    batch = lm.LossMaskBatch(len(frames), 4096, 512, 300 * 4)
    batch.stage(frames)
    batch.launch()
    grids = batch.results()
    wire = batch.wire.cpu().numpy()
    for j, g in enumerate(grids):
        want = np.packbits(g.reshape(-1))
        assert np.array_equal(wire[j, :len(want)], want)


def test_codec_tail_rule_and_explicit_ranges():
    lm = _lm()
    off = {k: LMASK["x_" + k + "_off"] for k in ("header", "ranges", "grid")}
    for i in range(len(LMASK["x_received_len"])):
        hdr = LMASK["x_header"][off["header"][i]:off["header"][i + 1]].tobytes()
        rng = LMASK["x_ranges"][off["ranges"][i]:off["ranges"][i + 1]].reshape(-1, 2)
        want = LMASK["x_grid"][off["grid"][i]:off["grid"][i + 1]].astype(bool)
        g = lm.decode_mask(hdr, int(LMASK["x_received_len"][i]), [tuple(r) for r in rng])
        assert np.array_equal(g.reshape(-1), want)


def test_random_headers_vs_oracle():
    """Synthetic headers incl. inverted/empty block ranges (malformed offsets)
    and every loss pattern density: kernel == oracle, bit for bit."""
    lm = _lm()
    from tools.synth import p_frame_header, n_data_shards
    rng = np.random.default_rng(77)
    frames, want = [], []
    for trial in range(300):
        w, h = [(64, 48), (320, 240), (1280, 720)][trial % 3]
        c = 3 if trial % 2 else 1
        L = 1024 if c == 3 else 512
        hdr, plen = p_frame_header(rng, w, h, c, present_ratio=rng.uniform(0, 0.5))
        if trial % 7 == 0 and len(hdr) > 14 + 8:
            # scramble offsets: inverted and empty ranges
            nblk = (w // 16) * (h // 16)
            o = 14 + (nblk + 7) // 8
            n_present = struct.unpack_from("<H", hdr, 12)[0]
            offs = np.frombuffer(hdr, "<u4", n_present, o).copy()
            rng.shuffle(offs)
            hdr = hdr[:o] + offs.tobytes()
        nd = n_data_shards(plen, L) + int(rng.integers(0, 3))
        recv = rng.random(nd) >= rng.choice([0.0, 0.05, 0.3, 1.0])
        recv[0] = True
        enc_len = len(hdr) + plen
        frames.append(lm.PFrameShards(hdr, nd, recv, L, enc_len))
        want.append(om.mask_from_shards(hdr, nd, {i for i in range(nd) if recv[i]}, L,
                                        enc_len))
    got = lm.loss_masks(frames)
    for g, wnt in zip(got, want):
        assert np.array_equal(g, wnt)


def test_undecodable_headers_raise():
    lm = _lm()
    good, plen = None, None
    from tools.synth import p_frame_header
    good, plen = p_frame_header(np.random.default_rng(1), 64, 64, 1, 0.5)
    bad = [good[:10],                                          # truncated fixed part
           good[:6] + bytes([0]) + good[7:],                   # block 0
           good[:20],                                          # truncated bitmap/offsets
           good[:14] + bytes([good[14] ^ 0x80]) + good[15:]]   # popcount mismatch
    for hdr in bad:
        with pytest.raises(om.UndecodableError):
            om.decode_mask(hdr, plen, [])
        with pytest.raises(lm.UndecodableError):
            lm.decode_mask(hdr, plen, [])
