"""Oracle: restatement of the reference SSIM metric.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Reference: ``pkg/src/rgbdstream/metrics.py:21-72`` -- single-scale SSIM
with an 8x8 uniform window over fully interior window positions,
C1 = (0.01*255)^2, C2 = (0.03*255)^2, float64 throughout, tri-channel planes
averaged per channel.  The reference computes the window means with
``scipy.ndimage.uniform_filter`` (mode="constant") and then keeps only the
interior positions (metrics.py:49-59); an interior window never touches the
zero padding, so its mean is the plain 8x8 box mean, computed here from
float64 integral images (summation order differs from the separable filter
at the 1e-13 level).  Pinned against the reference itself by
``tests/golden/make_golden.py gen_ssim`` -> ``tests/golden/ssim_golden.npz``.
"""

from __future__ import annotations

import numpy as np

SSIM_WINDOW = 8                       # metrics.py:21
_C1 = (0.01 * 255) ** 2               # metrics.py:22
_C2 = (0.03 * 255) ** 2               # metrics.py:23


def _box_mean(x: np.ndarray, w: int) -> np.ndarray:
    """Mean of every fully interior w x w window (valid positions)."""
    ii = np.zeros((x.shape[0] + 1, x.shape[1] + 1), np.float64)
    ii[1:, 1:] = x.cumsum(0).cumsum(1)
    s = ii[w:, w:] - ii[:-w, w:] - ii[w:, :-w] + ii[:-w, :-w]
    return s / float(w * w)


def _ssim_single(a: np.ndarray, b: np.ndarray) -> float:
    """metrics.py:41-63."""
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    w = SSIM_WINDOW
    h, wd = a.shape
    if h < w or wd < w:
        raise ValueError("plane smaller than the %dx%d SSIM window" % (w, w))
    mu_a, mu_b = _box_mean(a, w), _box_mean(b, w)
    var_a = _box_mean(a * a, w) - mu_a * mu_a
    var_b = _box_mean(b * b, w) - mu_b * mu_b
    cov = _box_mean(a * b, w) - mu_a * mu_b
    num = (2 * mu_a * mu_b + _C1) * (2 * cov + _C2)
    den = (mu_a ** 2 + mu_b ** 2 + _C1) * (var_a + var_b + _C2)
    return float(np.mean(num / den))


def ssim(a: np.ndarray, b: np.ndarray) -> float:
    """metrics.py:66-72: u8 planes (h, w) or (h, w, c)."""
    if a.shape != b.shape:
        raise ValueError("shape mismatch %r vs %r" % (a.shape, b.shape))
    if a.ndim == 3:
        return float(np.mean([_ssim_single(a[..., c], b[..., c])
                              for c in range(a.shape[2])]))
    return _ssim_single(a, b)
