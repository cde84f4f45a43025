"""Shared test helpers: seeded weights and inputs that do not depend on the
reference package, so the golden fixtures generated in the build container
(``tests/golden/make_golden.py``) can be re-created bit-identically on the
GPU box, where ``/root/reference`` does not exist."""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle.nvrec_forward import Arch, state_keys  # noqa: E402

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def state_shapes(arch: Arch, channels: int) -> dict:
    d, T, p, L = arch.dim, arch.tubelet_t, arch.patch, arch.layers
    nt = arch.stack_len // T
    shapes = {"time_pos": (nt, d), "embed.weight": (d, channels + 1, T, p, p),
              "embed.bias": (d,)}
    for i in range(L):
        pre = "blocks.%d." % i
        for n in ("norm_s", "norm_t", "norm_m"):
            shapes[pre + n + ".weight"] = (d,)
            shapes[pre + n + ".bias"] = (d,)
        for a in ("attn_s", "attn_t"):
            shapes[pre + a + ".qkv.weight"] = (3 * d, d)
            shapes[pre + a + ".qkv.bias"] = (3 * d,)
            shapes[pre + a + ".proj.weight"] = (d, d)
            shapes[pre + a + ".proj.bias"] = (d,)
        shapes[pre + "mlp.0.weight"] = (4 * d, d)
        shapes[pre + "mlp.0.bias"] = (4 * d,)
        shapes[pre + "mlp.2.weight"] = (d, 4 * d)
        shapes[pre + "mlp.2.bias"] = (d,)
    shapes["norm.weight"] = (d,)
    shapes["norm.bias"] = (d,)
    shapes["head.weight"] = (T * p * p * channels, d)
    shapes["head.bias"] = (T * p * p * channels,)
    assert list(shapes) == state_keys(L) or set(shapes) == set(state_keys(L))
    return shapes


def make_state(arch: Arch, channels: int, seed: int, perturb: bool = True) -> dict:
    """Seeded random-init weights with torch's default init scale
    (U(-1/sqrt(fan_in), 1/sqrt(fan_in)) for conv/linear weights and biases,
    LN weight 1 / bias 0, time_pos 0).  ``perturb`` adds N(0, 0.02) to
    time_pos, LN affine and biases so indexing bugs cannot
    hide behind zeros and ones."""
    rng = np.random.default_rng(seed)
    out = {}
    for key, shape in state_shapes(arch, channels).items():
        if key == "time_pos":
            v = np.zeros(shape, np.float32)
        elif ".norm" in key or key.startswith("norm."):
            v = np.ones(shape, np.float32) if key.endswith("weight") \
                else np.zeros(shape, np.float32)
        else:
            wkey = key[:-4] + "weight" if key.endswith("bias") else key
            wshape = state_shapes(arch, channels)[wkey]
            fan_in = int(np.prod(wshape[1:]))
            bound = 1.0 / np.sqrt(fan_in)
            v = rng.uniform(-bound, bound, shape).astype(np.float32)
        if perturb and (key == "time_pos" or key.endswith("bias")
                        or ".norm" in key or key.startswith("norm.")):
            v = (v + rng.normal(0.0, 0.02, shape)).astype(np.float32)
        out[key] = v
    return {k: out[k] for k in state_keys(arch.layers)}


def rand_u8(rng, shape):
    return rng.integers(0, 256, shape, dtype=np.uint8)


def textured_u8(rng, n, h, w, c, cell=8):
    """Coarse-cell textures (like rgbdstream.synthetic._coarse) with a slow
    drift between frames; (n, h, w, c) uint8."""
    ch, cw = -(-h // cell) + 2, -(-w // cell) + 2
    tile = rng.integers(0, 256, (ch, cw, c), dtype=np.uint8)
    tex = np.kron(tile, np.ones((cell, cell, 1), np.uint8))
    out = []
    for i in range(n):
        dy, dx = (i * 1) % cell, (i * 2) % cell
        out.append(tex[dy:dy + h, dx:dx + w])
    return np.stack(out)


def block_grid(rng, gh, gw, ratio):
    """``nvrec.data.synthetic_mask`` grid (data.py:137-142)."""
    return rng.random((gh, gw)) < ratio


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()[:16]
