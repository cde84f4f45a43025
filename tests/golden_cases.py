"""Golden-case definitions shared by ``tests/golden/make_golden.py`` (which
runs the UNMODIFIED reference in the build container) and the tests (which
rebuild the same seeded inputs anywhere, including the GPU box).

Model cases exercise ``MaskedVideoModel.forward`` (model.py:82-122) with
float stacks and arbitrary pixel masks; recover cases exercise
``RecoveryServer._recover`` (server.py:181-196) on u8 planes with block
grids.
"""

from __future__ import annotations

import numpy as np

from helpers import Arch, block_grid, make_state, textured_u8

DEFAULT = dict(k=5, tubelet_t=2, patch=16, dim=64, layers=2, heads=2)
SMALL = dict(k=2, tubelet_t=1, patch=16, dim=16, layers=1, heads=2)

# name -> (arch kwargs, channels, b, f, h, w, mask kind, seed)
MODEL_CASES = {
    "m_rgb_48x64_b2": (DEFAULT, 3, 2, 6, 48, 64, "blocks", 11),
    "m_depth_48x64_pad": (DEFAULT, 1, 1, 3, 48, 64, "pixels", 12),
    "m_rgb_96x128": (DEFAULT, 3, 1, 6, 96, 128, "pixels", 13),
    "m_depth_128x256_onetile": (DEFAULT, 1, 1, 6, 128, 256, "blocks", 14),
    "m_depth_240x320": (DEFAULT, 1, 1, 6, 240, 320, "blocks", 15),
    "m_small_rgb_32x48": (SMALL, 3, 2, 3, 32, 48, "pixels", 16),
    "m_k7_t2_depth": (dict(DEFAULT, k=7, dim=16), 1, 1, 8, 32, 32, "pixels", 17),
    "m_k3_t1_rgb": (dict(DEFAULT, k=3, tubelet_t=1, dim=32, heads=4), 3, 1, 4,
                    32, 64, "blocks", 18),
    "m_allmasked_16x16": (DEFAULT, 1, 1, 2, 16, 16, "all", 19),
    "m_nomask_rgb_32x32": (DEFAULT, 3, 1, 6, 32, 32, "none", 20),
}

# name -> (channels, n_refs, h, w, mask ratio, seed)
RECOVER_CASES = {
    "r_rgb_240x320_k5": (3, 5, 240, 320, 0.10, 31),
    "r_depth_240x320_k3": (1, 3, 240, 320, 0.10, 32),
    "r_rgb_96x128_k7refs": (3, 7, 96, 128, 0.30, 33),   # more refs than k
    "r_depth_48x64_k1": (1, 1, 48, 64, 0.25, 34),
}


def model_case(name):
    arch_kw, c, b, f, h, w, mkind, seed = MODEL_CASES[name]
    arch = Arch(**arch_kw)
    rng = np.random.default_rng(seed)
    state = make_state(arch, c, seed + 1000)
    stack = rng.random((b, f, c, h, w), dtype=np.float32)
    if mkind == "blocks":
        g = block_grid(rng, b * (h // 16), w // 16, 0.3).reshape(b, h // 16, w // 16)
        mask = np.repeat(np.repeat(g, 16, 1), 16, 2)
    elif mkind == "pixels":
        mask = rng.random((b, h, w)) < 0.2
        mask[:, : h // 2, : w // 4] = True      # a partial-patch hole
    elif mkind == "all":
        mask = np.ones((b, h, w), bool)
    else:
        mask = np.zeros((b, h, w), bool)
    return arch, c, state, stack, mask


def recover_case(name):
    c, nref, h, w, ratio, seed = RECOVER_CASES[name]
    arch = Arch(**DEFAULT)
    rng = np.random.default_rng(seed)
    state = make_state(arch, c, seed + 1000)
    frames = textured_u8(rng, nref + 1, h, w, c)
    grid = block_grid(rng, h // 16, w // 16, ratio)
    if not grid.any():
        grid[0, 0] = True
    plane = frames[-1].copy()
    pix = np.repeat(np.repeat(grid, 16, 0), 16, 1)
    plane[pix] = 0                          # zero-filled decode output
    refs = [frames[i] for i in range(nref)]
    return arch, c, state, plane, grid, refs


# name -> (channels, h, w, mask ratio, seed, n_refs) for recover_baseline
# (rgbdstream/recovery.py:128-196); dense masks exercise fully-masked rings
BASELINE_CASES = {
    "b_rgb_48x64": (3, 48, 64, 0.3, 41, 2),
    "b_rgb_96x128_dense": (3, 96, 128, 0.7, 42, 1),
    "b_rgb_240x320": (3, 240, 320, 0.1, 43, 5),
    "b_depth_48x64": (1, 48, 64, 0.3, 44, 2),
    "b_depth_96x128_dense": (1, 96, 128, 0.7, 45, 3),
    "b_depth_240x320": (1, 240, 320, 0.1, 46, 5),
    "b_depth_16x16_all": (1, 16, 16, 1.0, 47, 1),
}


def baseline_case(name):
    c, h, w, ratio, seed, nref = BASELINE_CASES[name]
    rng = np.random.default_rng(seed)
    frames = textured_u8(rng, nref + 1, h, w, c)
    if c == 1:
        frames = frames[..., 0]
    grid = block_grid(rng, h // 16, w // 16, ratio)
    if not grid.any():
        grid[0, 0] = True
    plane = frames[-1].copy()
    pix = np.repeat(np.repeat(grid, 16, 0), 16, 1)
    plane[pix] = 0
    return c, plane, grid, [frames[i] for i in range(nref)]


# name -> (shape, noise std, seed) for the SSIM metric (rgbdstream
# metrics.py:41-72): a textured plane against a noisy / shifted copy
SSIM_CASES = {
    "s_rgb_240x320_noise": ((240, 320, 3), 12.0, 51),
    "s_depth_240x320_noise": ((240, 320), 4.0, 52),
    "s_rgb_48x64_heavy": ((48, 64, 3), 60.0, 53),
    "s_depth_17x23_odd": ((17, 23), 8.0, 54),
    "s_depth_8x8_min": ((8, 8), 20.0, 55),
    "s_rgb_32x32_identical": ((32, 32, 3), 0.0, 56),
    "s_depth_720x1280_noise": ((720, 1280), 3.0, 57),
}


def ssim_case(name):
    shape, std, seed = SSIM_CASES[name]
    rng = np.random.default_rng(seed)
    c = shape[2] if len(shape) == 3 else 1
    a = textured_u8(rng, 1, shape[0], shape[1], c)[0]
    if len(shape) == 2:
        a = a[..., 0]
    noise = rng.normal(0.0, std, a.shape) if std else 0.0
    b = np.clip(np.rint(a.astype(np.float64) + noise), 0, 255).astype(np.uint8)
    return a, b


def recover_truth(name):
    """The uncorrupted last frame of ``recover_case(name)`` (SSIM reference)."""
    c, nref, h, w, ratio, seed = RECOVER_CASES[name]
    rng = np.random.default_rng(seed)           # same draws as recover_case
    return textured_u8(rng, nref + 1, h, w, c)[-1]
