"""GPU drop-in for the reference's timeout / fault fallback
``rgbdstream.recovery.recover_baseline`` (recovery.py:128-196), bit-exact:
+-8 px SAD block match on the intact border ring against the most recent
reference, plus the 3x3 boundary median for depth (``nvrec_baseline_u8``)."""

from __future__ import annotations

import ctypes
import time

import numpy as np
import torch

from . import _native
from .backend import RecoveryResponse
from .recovery import pack_grid


def baseline_device(planes: torch.Tensor, refs: torch.Tensor, mask_bits: torch.Tensor,
                    depth: bool, out: torch.Tensor | None = None) -> torch.Tensor:
    """planes/refs: u8 (b, h, w, c) device (refs = each stream's most recent
    reference); mask_bits: u8 (b, ceil(gh*gw/8)).  Returns u8 (b, h, w, c)."""
    lib = _native.load_library()
    b, h, w, c = planes.shape
    need = lib.nvrec_baseline_workspace_bytes(b, h, w, c)
    if need < 0:
        _native.check(int(need))
    ws = torch.empty(int(need), dtype=torch.uint8, device=planes.device)
    if out is None:
        out = torch.empty_like(planes)
    _native.check(lib.nvrec_baseline_u8(int(depth), b, h, w, c, planes.data_ptr(),
                                        refs.data_ptr(), mask_bits.data_ptr(), out.data_ptr(),
                                        ws.data_ptr(), ws.numel(), _native.stream_ptr()))
    return out


def recover_baseline(req) -> RecoveryResponse:
    """``rgbdstream.recovery.recover_baseline`` semantics for one request."""
    t0 = time.perf_counter()
    plane = req.plane
    grid = np.asarray(req.mask.grid, bool)
    if not req.references:
        return RecoveryResponse(plane.copy(), (time.perf_counter() - t0) * 1e3, fallback=True)
    if not grid.any():
        return RecoveryResponse(plane.copy(), (time.perf_counter() - t0) * 1e3)
    dev = _native.require_cuda()
    p3 = plane if plane.ndim == 3 else plane[:, :, None]
    ref = np.asarray(req.references[-1])
    r3 = ref if ref.ndim == 3 else ref[:, :, None]
    depth = int(req.modality) != 0
    planes = torch.from_numpy(np.ascontiguousarray(p3)[None]).to(dev)
    refs = torch.from_numpy(np.ascontiguousarray(r3)[None]).to(dev)
    bits = torch.from_numpy(pack_grid(grid)[None]).to(dev)
    out = baseline_device(planes, refs, bits, depth)[0].cpu().numpy()
    out = out if plane.ndim == 3 else out[:, :, 0]
    return RecoveryResponse(out, (time.perf_counter() - t0) * 1e3)
