"""ctypes binding of ``libnvrec_b200.so`` (C-ABI in ``include/nvrec_b200.h``).

The product path has no CPU fallback: importing this module without the
built library, or calling it without a CUDA device, raises.  Buffers cross
the boundary as raw device pointers of torch tensors; launches go to the
caller's current CUDA stream (capture-safe: nothing here allocates or
synchronises on the hot path once the workspace for a shape exists).
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# NVREC_LIB: an alternative in-tree build of the same library (trace /
# experiment variants, tools/); the default is the product build
LIB_PATH = os.environ.get("NVREC_LIB") or os.path.join(_HERE, "lib", "libnvrec_b200.so")

PREC_FAST = 0
PREC_PRECISE = 1
_PREC = {"fast": PREC_FAST, "precise": PREC_PRECISE}

E_INVALID, E_UNSUPPORTED, E_CUDA, E_WORKSPACE, E_STATE = -1, -2, -3, -4, -5

EXPORTS = ("nvrec_abi_version", "nvrec_last_error", "nvrec_model_create",
           "nvrec_model_destroy", "nvrec_model_load", "nvrec_workspace_bytes",
           "nvrec_forward_f32", "nvrec_recover_u8", "nvrec_recover_u16", "nvrec_loss_mask",
           "nvrec_profile_begin", "nvrec_profile_end", "nvrec_baseline_workspace_bytes",
           "nvrec_baseline_u8", "nvrec_decode", "nvrec_rs_plan", "nvrec_rs_reconstruct",
           "nvrec_attn_fixup_items")
STAGES = ("lossmask", "masklist", "copy", "embed", "ln_qkv", "attn_simt", "attn_tc",
          "token", "baseline", "decode", "rs", "last_tc")
ABI_VERSION = 5


class NativeError(RuntimeError):
    """A non-argument failure inside libnvrec_b200 (CUDA, state, config)."""


class _Config(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("tubelet_t", ctypes.c_int32),
                ("patch", ctypes.c_int32), ("dim", ctypes.c_int32),
                ("layers", ctypes.c_int32), ("heads", ctypes.c_int32)]


class LossMaskJob(ctypes.Structure):
    """``nvrec_lossmask_job`` (device-pointer descriptor)."""
    _fields_ = [("header", ctypes.c_void_p), ("header_len", ctypes.c_int32),
                ("n_data", ctypes.c_int32), ("received", ctypes.c_void_p),
                ("shard_len", ctypes.c_int32), ("body_len", ctypes.c_int64),
                ("payload_received", ctypes.c_int64),
                ("extra_ranges", ctypes.c_void_p), ("n_extra", ctypes.c_int32),
                ("grid", ctypes.c_void_p), ("wire_bits", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("grid_capacity", ctypes.c_int32)]


class DecodeJob(ctypes.Structure):
    """``nvrec_decode_job``."""
    _fields_ = [("mask", LossMaskJob), ("payload", ctypes.c_void_p),
                ("reference", ctypes.c_void_p), ("plane", ctypes.c_void_p),
                ("plane_capacity", ctypes.c_int64), ("scratch", ctypes.c_void_p)]


class RsJob(ctypes.Structure):
    """``nvrec_rs_job``."""
    _fields_ = [("data", ctypes.c_void_p), ("parity", ctypes.c_void_p),
                ("coef", ctypes.c_void_p), ("sources", ctypes.c_void_p),
                ("missing", ctypes.c_void_p), ("n", ctypes.c_int32),
                ("r", ctypes.c_int32), ("m", ctypes.c_int32),
                ("shard_len", ctypes.c_int32)]


_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the shared library; raise if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                "libnvrec_b200.so not built (%s); run "
                "`python -c 'import __graft_entry__ as g; g.build()'` -- there is "
                "no CPU fallback for the nvrec B200 path" % path)
        lib = ctypes.CDLL(path)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        lib.nvrec_abi_version.restype = ctypes.c_int
        lib.nvrec_last_error.restype = ctypes.c_char_p
        lib.nvrec_model_create.argtypes = [ctypes.POINTER(_Config), i32,
                                           ctypes.POINTER(vp)]
        lib.nvrec_model_destroy.argtypes = [vp]
        lib.nvrec_model_load.argtypes = [vp, ctypes.POINTER(vp),
                                         ctypes.POINTER(i64), i32]
        lib.nvrec_workspace_bytes.argtypes = [vp, i32, i32, i32, i32]
        lib.nvrec_workspace_bytes.restype = i64
        lib.nvrec_forward_f32.argtypes = [vp, vp, i32, i32, i32, i32, i32, vp, vp,
                                          vp, i64, i32, vp]
        lib.nvrec_recover_u8.argtypes = [vp, i32, i32, i32, vp, i32, vp, vp, vp, vp,
                                         i64, i32, vp]
        lib.nvrec_recover_u16.argtypes = [vp, i32, i32, i32, vp, i32, vp, vp, vp, vp,
                                         i64, i32, vp]
        lib.nvrec_loss_mask.argtypes = [vp, i32, vp]
        lib.nvrec_baseline_workspace_bytes.argtypes = [i32, i32, i32, i32]
        lib.nvrec_baseline_workspace_bytes.restype = i64
        lib.nvrec_baseline_u8.argtypes = [i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, i64, vp]
        lib.nvrec_decode.argtypes = [vp, i32, i32, vp]
        lib.nvrec_rs_plan.argtypes = [i32, i32, vp, vp, vp, vp, ctypes.POINTER(i32)]
        lib.nvrec_rs_reconstruct.argtypes = [vp, i32, i32, i32, i32, vp]
        lib.nvrec_attn_fixup_items.restype = i64
        lib.nvrec_profile_end.argtypes = [ctypes.POINTER(ctypes.c_float),
                                          ctypes.POINTER(i32), i32]
        for name in EXPORTS:
            getattr(lib, name)
        if lib.nvrec_abi_version() != ABI_VERSION:
            raise RuntimeError("libnvrec_b200 ABI mismatch")
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load_library().nvrec_last_error().decode(errors="replace")
    if rc == E_INVALID:
        raise ValueError(msg)
    raise NativeError("nvrec_b200 error %d: %s" % (rc, msg))


def precision_code(p) -> int:
    if isinstance(p, int):
        return p
    try:
        return _PREC[p]
    except KeyError:
        raise ValueError("precision must be 'fast' or 'precise'") from None


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("nvrec_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device() if device is None
                        else torch.device(device).index or 0)


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class NativeModel:
    """Owns one ``nvrec_model`` (packed weights resident on one device) and a
    per-stream workspace cache."""

    def __init__(self, arch, channels: int, device: torch.device):
        lib = load_library()
        self.lib = lib
        self.device = device
        self.channels = channels
        cfg = _Config(arch.k, arch.tubelet_t, arch.patch, arch.dim, arch.layers,
                      arch.heads)
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            check(lib.nvrec_model_create(ctypes.byref(cfg), channels, ctypes.byref(h)))
        self.handle = h
        self._ws = {}

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib is not None:
            _lib.nvrec_model_destroy(h)
            self.handle = None

    def load(self, tensors) -> None:
        """fp32 state-dict tensors in ``MaskedVideoModel`` order."""
        host = [t.detach().to("cpu", torch.float32).contiguous() for t in tensors]
        ptrs = (ctypes.c_void_p * len(host))(*[t.data_ptr() for t in host])
        numel = (ctypes.c_int64 * len(host))(*[t.numel() for t in host])
        with torch.cuda.device(self.device):
            check(self.lib.nvrec_model_load(self.handle, ptrs, numel, len(host)))

    def workspace(self, b: int, h: int, w: int, prec: int) -> torch.Tensor:
        need = self.lib.nvrec_workspace_bytes(self.handle, b, h, w, prec)
        if need < 0:
            check(int(need))
        # per (stream, thread): two threads enqueueing on one stream would
        # otherwise interleave their launches over a shared workspace
        key = (stream_ptr(), threading.get_ident())
        ws = self._ws.get(key)
        if ws is None or ws.numel() < need:
            ws = torch.empty(int(need), dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def forward_f32(self, stack: torch.Tensor, mask: torch.Tensor, prec: int) -> torch.Tensor:
        b, f, c, h, w = stack.shape
        out = torch.empty((b, c, h, w), dtype=torch.float32, device=self.device)
        ws = self.workspace(b, h, w, prec)
        check(self.lib.nvrec_forward_f32(self.handle, stack.data_ptr(), b, f, c, h, w,
                                         mask.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                         ws.numel(), prec, stream_ptr()))
        return out

    def recover_u8(self, frames: torch.Tensor, frame_index: torch.Tensor,
                   mask_bits: torch.Tensor, out: torch.Tensor | None, b: int, h: int, w: int,
                   prec: int) -> torch.Tensor | None:
        """out=None merges in place into each stream's corrupted-plane slot."""
        ws = self.workspace(b, h, w, prec)
        check(self.lib.nvrec_recover_u8(self.handle, b, h, w, frames.data_ptr(),
                                        frames.shape[0], frame_index.data_ptr(), mask_bits.data_ptr(),
                                        None if out is None else out.data_ptr(),
                                        ws.data_ptr(), ws.numel(), prec, stream_ptr()))
        return out


    def recover_u16(self, frames: torch.Tensor, frame_index: torch.Tensor,
                    mask_bits: torch.Tensor, out: torch.Tensor | None, b: int, h: int, w: int,
                    prec: int) -> torch.Tensor | None:
        """16-bit depth planes (n_slots, h, w) uint16; out=None merges in place."""
        ws = self.workspace(b, h, w, prec)
        check(self.lib.nvrec_recover_u16(self.handle, b, h, w, frames.data_ptr(),
                                         frames.shape[0], frame_index.data_ptr(),
                                         mask_bits.data_ptr(),
                                         None if out is None else out.data_ptr(),
                                         ws.data_ptr(), ws.numel(), prec, stream_ptr()))
        return out


def attn_fixup_items() -> int:
    """Attention work items recomputed by the exact fix-up so far (device-wide
    counter, current device)."""
    n = load_library().nvrec_attn_fixup_items()
    if n < 0:
        check(int(n))
    return int(n)


class StageProfile:
    """Context manager around ``nvrec_profile_begin/end``: per-stage device
    milliseconds and launch counts of every library kernel launched inside."""

    def __enter__(self):
        check(load_library().nvrec_profile_begin())
        return self

    def __exit__(self, *exc):
        n = len(STAGES)
        ms = (ctypes.c_float * n)()
        cnt = (ctypes.c_int32 * n)()
        total = load_library().nvrec_profile_end(ms, cnt, n)
        if total < 0:
            check(total)
        self.ms = {STAGES[i]: float(ms[i]) for i in range(n)}
        self.launches = {STAGES[i]: int(cnt[i]) for i in range(n)}
        self.total_launches = int(total)
        return False
