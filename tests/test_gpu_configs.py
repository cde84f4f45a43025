"""BASELINE.json configurations as parity cases (the bench runs configs[2]
x configs[4]; these cover the others against the CPU oracle):

  configs[0]  single 320x240 RGB-D frame, 10% loss           (also golden)
  configs[1]  640x480 RGB + 16-bit depth, 30-frame sequence, Bernoulli 5%
  configs[3]  1920x1080 (padded to 1088, frames.py:101-109) RGB-D, 20% loss
"""

import numpy as np
import pytest
import torch

from helpers import block_grid, make_state, textured_u8
from oracle import nvrec_forward, recover as oracle_recover

pytestmark = pytest.mark.gpu

ARCH = nvrec_forward.Arch()


def _model(c, seed, precision):
    from paper_2604_27441_b200 import MaskedVideoModel, ModelConfig
    st = make_state(ARCH, c, seed)
    m = MaskedVideoModel(ModelConfig(), c, precision=precision)
    m.load_state_dict({k: torch.from_numpy(v) for k, v in st.items()})
    return m, st


def _pad16(a):
    h, w = a.shape[-3:-1] if a.ndim == 4 else a.shape[-2:]
    ph, pw = (-h) % 16, (-w) % 16
    pads = [(0, 0)] * (a.ndim - 3 if a.ndim == 4 else a.ndim - 2) + [(0, ph), (0, pw)]
    if a.ndim == 4:
        pads.append((0, 0))
    return np.pad(a, pads, mode="edge")          # rgbdstream.frames.pad_to_block


@pytest.mark.parametrize("c", [3, 1])
def test_config0_320x240_single_frame(c):
    from paper_2604_27441_b200.recovery import RecoveryEngine
    rng = np.random.default_rng(100 + c)
    m, st = _model(c, 1000 + c, "fast")
    frames = textured_u8(rng, 6, 240, 320, c)
    grid = block_grid(rng, 15, 20, 0.10)
    grid[0, 0] = True
    got = RecoveryEngine(m, "fast").recover(frames[-1], grid, list(frames[:-1]))
    want = oracle_recover.recover(st, ARCH, c, frames[-1], grid, list(frames[:-1]))
    assert np.abs(got.astype(int) - want.astype(int)).max() <= 2


def test_config1_640x480_rgb_and_depth16_sequence():
    """30-frame sequence: recovered frames join the ring (receiver.py:268-269);
    RGB on the fast u8 path (<= 2 LSB), 16-bit depth on the precise float path
    (<= 1 depth unit, i.e. <= 1 mm at 1 mm/unit)."""
    from paper_2604_27441_b200.recovery import RecoveryEngine, recover_depth16
    rng = np.random.default_rng(7)
    mr, str_ = _model(3, 1103, "fast")
    md, std = _model(1, 1101, "precise")
    eng = RecoveryEngine(mr, "fast")
    rgb = textured_u8(rng, 35, 480, 640, 3)
    base = rng.integers(200, 4000, (480 // 8 + 2, 640 // 8 + 2)).astype(np.uint16)
    depth = np.stack([np.kron(base, np.ones((8, 8), np.uint16))[i % 8:i % 8 + 480, :640]
                      + np.uint16(i) for i in range(35)])
    ring_r = [rgb[i] for i in range(5)]
    ring_d_gpu = [depth[i] for i in range(5)]
    ring_d_ref = [depth[i] for i in range(5)]
    worst_r, worst_d = 0, 0
    for t in range(5, 35):
        grid = block_grid(rng, 30, 40, 0.05)
        grid[t % 30, t % 40] = True
        pr = rgb[t].copy()
        got = eng.recover(pr, grid, ring_r)
        want = oracle_recover.recover(str_, ARCH, 3, pr, grid, ring_r)
        worst_r = max(worst_r, int(np.abs(got.astype(int) - want.astype(int)).max()))
        ring_r = ring_r[1:] + [want]              # both sides continue from the reference
        gd = recover_depth16(md, depth[t], grid, ring_d_gpu)
        # oracle: same 16-bit normalisation through the fp32 reference forward
        stack = np.stack(ring_d_ref[-5:] + [depth[t]]).astype(np.float32) / 65535.0
        pix = np.repeat(np.repeat(grid, 16, 0), 16, 1)
        out = nvrec_forward.forward(std, ARCH, 1, stack[None, :, None], pix[None]).numpy()[0, 0]
        q = np.clip(out * 65535.0 + 0.5, 0, 65535).astype(np.uint16)
        wd = np.where(pix, q, depth[t])
        worst_d = max(worst_d, int(np.abs(gd.astype(int) - wd.astype(int)).max()))
        ring_d_gpu = ring_d_gpu[1:] + [gd]
        ring_d_ref = ring_d_ref[1:] + [wd]
    assert worst_r <= 2, worst_r
    assert worst_d <= 1, worst_d


@pytest.mark.parametrize("c", [3, 1])
def test_config3_1080p_padded_20pct(c):
    from paper_2604_27441_b200.recovery import RecoveryEngine
    rng = np.random.default_rng(300 + c)
    m, st = _model(c, 1300 + c, "fast")
    frames = _pad16(textured_u8(rng, 6, 1080, 1920, c))
    assert frames.shape[1:3] == (1088, 1920)
    grid = block_grid(rng, 68, 120, 0.20)
    got = RecoveryEngine(m, "fast").recover(frames[-1], grid, list(frames[:-1]))
    want = oracle_recover.recover(st, ARCH, c, frames[-1], grid, list(frames[:-1]))
    assert np.abs(got.astype(int) - want.astype(int)).max() <= 2
