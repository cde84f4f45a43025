"""``MaskedVideoModel`` -- drop-in for ``nvrec.model.MaskedVideoModel``.

Same constructor, parameter names/shapes/initialisation (so
``torch.manual_seed(s); MaskedVideoModel(cfg, c)`` yields the reference's
weights and ``load_state_dict`` accepts reference checkpoints), same forward
contract and ``ValueError`` messages (reference model.py:67-122).  The
forward itself runs in ``libnvrec_b200.so`` on the GPU: the nn submodules
below are parameter containers only and are never called.

Inference only: the returned tensor carries no autograd graph (training is
outside the recovery path).
"""

from __future__ import annotations

import threading

import torch
from torch import nn

from . import _native
from .config import ModelConfig


class _Attention(nn.Module):
    """Parameter container of reference ``_Attention`` (model.py:27-32)."""

    def __init__(self, dim: int, heads: int):
        super().__init__()
        self.heads = heads
        self.qkv = nn.Linear(dim, dim * 3)
        self.proj = nn.Linear(dim, dim)


class _Block(nn.Module):
    """Parameter container of reference ``_Block`` (model.py:43-54)."""

    def __init__(self, dim: int, heads: int):
        super().__init__()
        self.norm_s = nn.LayerNorm(dim)
        self.attn_s = _Attention(dim, heads)
        self.norm_t = nn.LayerNorm(dim)
        self.attn_t = _Attention(dim, heads)
        self.norm_m = nn.LayerNorm(dim)
        self.mlp = nn.Sequential(nn.Linear(dim, dim * 4), nn.GELU(),
                                 nn.Linear(dim * 4, dim))


class MaskedVideoModel(nn.Module):
    """Masked-video reconstruction transformer (reference model.py:67-80).

    ``precision``: ``"fast"`` (bf16 tensor-core attention, fp32 elsewhere;
    RGB and 8-bit depth) or ``"precise"`` (fp32 throughout; 16-bit depth)."""

    def __init__(self, config: ModelConfig, channels: int, precision: str = "fast"):
        super().__init__()
        self.config = config
        self.channels = channels
        self.precision = precision
        t, p, d = config.tubelet_t, config.patch, config.dim
        # registration order == reference (state-dict order, init RNG order)
        self.embed = nn.Conv3d(channels + 1, d, kernel_size=(t, p, p), stride=(t, p, p))
        self.time_pos = nn.Parameter(torch.zeros(config.stack_len // t, d))
        self.blocks = nn.ModuleList(_Block(d, config.heads) for _ in range(config.layers))
        self.norm = nn.LayerNorm(d)
        self.head = nn.Linear(d, t * p * p * channels)
        self._native = None
        self._packed_sig = None
        self._native_lock = threading.Lock()

    # -- weights -> device ----------------------------------------------------

    def _signature(self):
        # parameters are stable objects: in-place updates (load_state_dict,
        # optimiser steps) bump _version, re-assignment changes data_ptr
        return tuple((v.data_ptr(), v._version) for v in self.parameters())

    def native(self, device=None) -> _native.NativeModel:
        """The packed on-device model, re-packed when any parameter changed."""
        dev = _native.require_cuda(device)
        sig = self._signature()
        nat = self._native
        if nat is not None and nat.device == dev and self._packed_sig == sig:
            return nat
        # serving threads share one model: create / re-pack exactly once
        with self._native_lock:
            if self._native is None or self._native.device != dev:
                self._native = _native.NativeModel(self.config, self.channels, dev)
                self._packed_sig = None
            if self._packed_sig != sig:
                self._native.load(list(self.state_dict().values()))
                self._packed_sig = sig
            return self._native

    def native_snapshot(self, device=None) -> _native.NativeModel:
        """A private packed copy of the current weights.  Serving pipelines
        capture CUDA graphs over the packed weight pointers, so they must not
        share the re-packable ``native()`` object: a later ``load_state_dict``
        followed by a module call would free the blob their graphs read."""
        dev = _native.require_cuda(device)
        nat = _native.NativeModel(self.config, self.channels, dev)
        nat.load(list(self.state_dict().values()))
        return nat

    # -- forward -------------------------------------------------------------

    def forward(self, stack: torch.Tensor, mask: torch.Tensor) -> torch.Tensor:
        """Reconstruct the last frame of ``stack`` (reference model.py:82-122).

        stack: (batch, frames, channels, h, w) in [0, 1], oldest first, the
        corrupted frame last (front-padded with the oldest frame when shorter
        than ``config.stack_len``); mask: (batch, h, w) bool, True where the
        last frame is corrupted.  Returns (batch, channels, h, w) float32 on
        the input's device."""
        cfg = self.config
        b, f, c, h, w = stack.shape
        if c != self.channels:
            raise ValueError("expected %d channels, got %d" % (self.channels, c))
        if h % cfg.patch or w % cfg.patch:
            raise ValueError("frame size must be a multiple of the patch edge")
        if f > cfg.stack_len:
            raise ValueError("stack longer than configured length")
        if tuple(mask.shape) != (b, h, w):
            raise ValueError("mask must have shape (batch, h, w)")
        nat = self.native(stack.device if stack.is_cuda else None)
        dev = nat.device
        with torch.cuda.device(dev):
            st = stack.detach().to(dev, torch.float32).contiguous()
            mk = mask.detach().to(dev)
            # bool and uint8 share the byte layout (nonzero = corrupted): no copy
            mk = (mk.view(torch.uint8) if mk.dtype == torch.bool else
                  mk if mk.dtype == torch.uint8 else (mk != 0).to(torch.uint8)).contiguous()
            out = nat.forward_f32(st, mk, _native.precision_code(self.precision))
        return out if stack.is_cuda else out.to(stack.device)
