"""In-process recovery backend with a device-resident reference ring.

Drop-in for the receiver's backend callable (reference
``rgbdstream/receiver.py:90-100,260-264``: ``backend(RecoveryRequest) ->
RecoveryResponse``) -- the cheapest integration of the B200 path: no TCP,
no per-request re-upload of the k references.

The receiver's ``ReferenceRing`` (recovery.py:64-83) hands every request
the same numpy plane objects it already showed us (recovered planes it got
back from this backend, or clean decodes it pushed in between).  The
backend keeps a small identity-keyed cache of device copies of those planes
(holding a reference to each host array, so an id cannot be recycled while
cached), so in steady state a request uploads only its new corrupted plane;
the recovered plane is written on the device and its device copy is cached
under the returned host array, ready to be a reference of the next request.

Semantics match the remote path (server.py:181-196 + recovery.py:347):
echo for an empty mask / no references / a modality without a model, and
trusted pixels are never rewritten.
"""

from __future__ import annotations

import time
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .checkpoint import Checkpoint
from .data import MOD_DEPTH, MOD_RGB
from .recovery import RecoveryEngine, pack_grid, stack_slots


@dataclass
class RecoveryResponse:
    """Field-compatible with ``rgbdstream.recovery.RecoveryResponse``
    (recovery.py:56-61)."""
    plane: np.ndarray
    latency_ms: float
    fallback: bool = False
    timeout: bool = False


class _PlaneCache:
    """id(host array) -> (host array, device plane), LRU-bounded."""

    def __init__(self, capacity: int):
        self.capacity = capacity
        self.items: OrderedDict[int, tuple] = OrderedDict()
        self.uploads = 0

    def get(self, host: np.ndarray, device, shape):
        key = id(host)
        hit = self.items.get(key)
        if hit is not None and hit[0] is host:
            self.items.move_to_end(key)
            return hit[1]
        dev = torch.from_numpy(np.ascontiguousarray(host).reshape(shape)).to(
            device, non_blocking=True)
        self.uploads += 1
        self.put(host, dev)
        return dev

    def put(self, host: np.ndarray, dev: torch.Tensor):
        self.items[id(host)] = (host, dev)
        self.items.move_to_end(id(host))
        while len(self.items) > self.capacity:
            self.items.popitem(last=False)


class B200Backend:
    """``backend(req) -> RecoveryResponse`` for ``rgbdstream.receiver.Receiver``.

    ``checkpoint_rgb`` / ``checkpoint_depth``: ``Checkpoint`` objects (either
    this package's or the reference's -- same fields)."""

    def __init__(self, checkpoint_rgb=None, checkpoint_depth=None,
                 precision_rgb: str = "fast", precision_depth: str = "fast",
                 device=None, cache_planes: int = 16):
        self.device = _native.require_cuda(device)
        self.engines = {}
        self.caches = {}
        for mod, ck, prec in ((MOD_RGB, checkpoint_rgb, precision_rgb),
                              (MOD_DEPTH, checkpoint_depth, precision_depth)):
            if ck is None:
                continue
            ck = Checkpoint(config=ck.config, channels=ck.channels, state=ck.state)
            self.engines[mod] = RecoveryEngine(ck.build_model(precision=prec), prec)
            self.caches[mod] = _PlaneCache(cache_planes)
        self.stream = torch.cuda.Stream(self.device)

    def __call__(self, req) -> RecoveryResponse:
        t0 = time.perf_counter()
        mod = int(req.modality)
        plane = req.plane
        grid = np.asarray(req.mask.grid, bool)
        refs = list(req.references)
        eng = self.engines.get(mod)
        if eng is None or not refs or not grid.any():
            return RecoveryResponse(plane.copy(), (time.perf_counter() - t0) * 1e3,
                                    fallback=not refs)
        cfg = eng.model.config
        h, w = plane.shape[:2]
        c = eng.channels
        shape = (h, w, c)
        cache = self.caches[mod]
        refs = refs[-cfg.k:]
        with torch.cuda.stream(self.stream):
            dev_refs = [cache.get(r, self.device, shape) for r in refs]
            dev_plane = torch.from_numpy(np.ascontiguousarray(plane).reshape(shape)).to(
                self.device, non_blocking=True)
            frames = torch.stack(dev_refs + [dev_plane])
            index = torch.tensor([stack_slots(len(refs), cfg.k, cfg.stack_len)],
                                 dtype=torch.int32).to(self.device, non_blocking=True)
            bits = torch.from_numpy(pack_grid(grid)[None]).to(self.device, non_blocking=True)
            out = eng.recover_device(frames, index, bits)
            host = torch.empty(out.shape[1:], dtype=torch.uint8, pin_memory=True)
            host.copy_(out[0], non_blocking=True)
        self.stream.synchronize()
        res = host.numpy()
        res = res if plane.ndim == 3 else res[:, :, 0]
        res = res.copy()
        cache.put(res, out[0])          # the receiver pushes this plane to its ring
        return RecoveryResponse(res, (time.perf_counter() - t0) * 1e3)
