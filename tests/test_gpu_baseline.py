"""GPU block-match fallback vs the reference's recover_baseline (golden,
bit-exact) and vs the oracle at 1280x720."""

import os
from dataclasses import dataclass

import numpy as np
import pytest

from golden_cases import BASELINE_CASES, baseline_case
from helpers import GOLDEN_DIR, block_grid, textured_u8
from oracle import baseline as ob

pytestmark = pytest.mark.gpu
BASE = np.load(os.path.join(GOLDEN_DIR, "baseline_golden.npz"))


@dataclass
class _Mask:
    grid: np.ndarray


@dataclass
class _Req:
    frame_id: int
    modality: int
    plane: np.ndarray
    mask: _Mask
    references: list


@pytest.mark.parametrize("name", sorted(BASELINE_CASES))
def test_gpu_baseline_matches_reference(name):
    from paper_2604_27441_b200.baseline import recover_baseline
    c, plane, grid, refs = baseline_case(name)
    resp = recover_baseline(_Req(1, 0 if c == 3 else 1, plane, _Mask(grid), refs))
    assert np.array_equal(resp.plane, BASE[name])


@pytest.mark.parametrize("c", [3, 1])
def test_gpu_baseline_720p_vs_oracle(c):
    from paper_2604_27441_b200.baseline import recover_baseline
    rng = np.random.default_rng(70 + c)
    frames = textured_u8(rng, 2, 720, 1280, c)
    if c == 1:
        frames = frames[..., 0]
    grid = block_grid(rng, 45, 80, 0.15)
    plane = frames[1].copy()
    plane[np.repeat(np.repeat(grid, 16, 0), 16, 1)] = 0
    resp = recover_baseline(_Req(1, 0 if c == 3 else 1, plane, _Mask(grid), [frames[0]]))
    want, _ = (ob.baseline_rgb if c == 3 else ob.baseline_depth)(plane, grid, [frames[0]])
    assert np.array_equal(resp.plane, want)


def test_gpu_baseline_fallback_rules():
    from paper_2604_27441_b200.baseline import recover_baseline
    plane = np.full((32, 32, 3), 5, np.uint8)
    r = recover_baseline(_Req(1, 0, plane, _Mask(np.ones((2, 2), bool)), []))
    assert r.fallback and np.array_equal(r.plane, plane)
    r = recover_baseline(_Req(1, 0, plane, _Mask(np.zeros((2, 2), bool)), [plane]))
    assert not r.fallback and np.array_equal(r.plane, plane)
