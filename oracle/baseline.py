"""Oracle: restatement of the reference's timeout/fault fallback
``recover_baseline`` (rgbdstream/recovery.py:94-196).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

* RGB (recovery.py:128-159): every masked 16-px block is replaced by the
  best-matching block of the most recent reference, found by a +-8 px shift
  search scored with SAD on the block's intact one-pixel border ring
  (``_ring_coords`` :94-106, ``_best_shift`` :109-125: score = SAD / #valid
  + 1e-6 * (|dy| + |dx|) in float64, first minimum in (dy, dx) raster order).
* Depth (recovery.py:162-184): the RGB result, then a 3x3 median (mode
  'nearest' on the masked bounding box +-2 px) applied on the two-pixel band
  straddling the mask boundary (4-connected binary dilation).
"""

from __future__ import annotations

import numpy as np
from scipy.ndimage import binary_dilation, median_filter

SEARCH_RADIUS = 8
BLOCK = 16


def ring_coords(y0, x0, block, h, w):
    """recovery.py:94-106 (order preserved)."""
    ys, xs = [], []
    for x in range(x0 - 1, x0 + block + 1):
        ys.extend((y0 - 1, y0 + block))
        xs.extend((x, x))
    for y in range(y0, y0 + block):
        ys.extend((y, y))
        xs.extend((x0 - 1, x0 + block))
    ys = np.asarray(ys)
    xs = np.asarray(xs)
    keep = (ys >= 0) & (ys < h) & (xs >= 0) & (xs < w)
    return ys[keep], xs[keep]


def best_shift(ty, tx, tvals, ref, rad=SEARCH_RADIUS):
    """recovery.py:109-125."""
    h, w = ref.shape[:2]
    shifts = np.arange(-rad, rad + 1)
    dys, dxs = np.meshgrid(shifts, shifts, indexing="ij")
    dys, dxs = dys.reshape(-1), dxs.reshape(-1)
    ys = ty[None, :] + dys[:, None]
    xs = tx[None, :] + dxs[:, None]
    valid = (ys >= 0) & (ys < h) & (xs >= 0) & (xs < w)
    cand = ref[np.clip(ys, 0, h - 1), np.clip(xs, 0, w - 1)].astype(np.int32)
    diff = np.abs(cand - tvals.astype(np.int32)[None])
    if diff.ndim == 3:
        diff = diff.sum(axis=-1)
    sad = np.where(valid, diff, 0).sum(axis=1).astype(np.float64)
    nvalid = valid.sum(axis=1)
    score = np.where(nvalid > 0, sad / np.maximum(nvalid, 1), np.inf)
    score += 1e-6 * (np.abs(dys) + np.abs(dxs))
    best = int(np.argmin(score))
    return int(dys[best]), int(dxs[best])


def baseline_rgb(plane, grid, refs):
    """recovery.py:128-159 -> (plane, fallback)."""
    if not refs:
        return plane.copy(), True
    if not grid.any():
        return plane.copy(), False
    ref = refs[-1]
    h, w = plane.shape[:2]
    out = plane.copy()
    pix = np.repeat(np.repeat(grid, BLOCK, 0), BLOCK, 1)
    for by, bx in zip(*np.nonzero(grid)):
        y0, x0 = by * BLOCK, bx * BLOCK
        ry, rx = ring_coords(y0, x0, BLOCK, h, w)
        intact = ~pix[ry, rx]
        if intact.any():
            ry, rx = ry[intact], rx[intact]
        else:
            yy, xx = np.meshgrid(np.arange(y0, y0 + BLOCK), np.arange(x0, x0 + BLOCK),
                                 indexing="ij")
            ry, rx = yy.reshape(-1), xx.reshape(-1)
        dy, dx = best_shift(ry, rx, plane[ry, rx], ref)
        sy = np.clip(np.arange(y0, y0 + BLOCK) + dy, 0, h - 1)
        sx = np.clip(np.arange(x0, x0 + BLOCK) + dx, 0, w - 1)
        out[y0:y0 + BLOCK, x0:x0 + BLOCK] = ref[np.ix_(sy, sx)]
    chans = 1 if plane.ndim == 2 else plane.shape[2]
    m = pix if chans == 1 else np.repeat(pix[:, :, None], chans, axis=2)
    return np.where(m, out, plane), False


def baseline_depth(plane, grid, refs):
    """recovery.py:162-184 (plane is (h, w))."""
    base, fb = baseline_rgb(plane, grid, refs)
    if fb or not grid.any():
        return base, fb
    pix = np.repeat(np.repeat(grid, BLOCK, 0), BLOCK, 1)
    ys, xs = np.nonzero(pix)
    h, w = base.shape[:2]
    y0, y1 = max(ys.min() - 2, 0), min(ys.max() + 3, h)
    x0, x1 = max(xs.min() - 2, 0), min(xs.max() + 3, w)
    sub = base[y0:y1, x0:x1]
    sp = pix[y0:y1, x0:x1]
    boundary = binary_dilation(sp) & ~sp | (binary_dilation(~sp) & sp)
    smoothed = median_filter(sub, size=3, mode="nearest")
    out = base.copy()
    out[y0:y1, x0:x1] = np.where(boundary, smoothed, sub)
    return out, False
