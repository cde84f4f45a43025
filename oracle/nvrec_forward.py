"""Oracle: functional CPU restatement of ``MaskedVideoModel.forward``.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Reference: ``pkg/nvrec/src/nvrec/model.py``.  Every step below cites the
line it restates.  The arithmetic is fp32 torch-CPU (``F.conv3d``,
``F.layer_norm``, ``F.linear``, ``F.scaled_dot_product_attention``,
``F.gelu``, ``torch.sigmoid``) -- the same ATen kernels the reference module
dispatches to, but written as plain functions over a state
dict so the oracle does not import the reference package.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F


@dataclass(frozen=True)
class Arch:
    """Architecture fields of ``ModelConfig`` (``config.py:14-19,35-41``)."""
    k: int = 5
    tubelet_t: int = 2
    patch: int = 16
    dim: int = 64
    layers: int = 2
    heads: int = 2

    @property
    def stack_len(self) -> int:          # config.py:35-41
        raw = self.k + 1
        return raw + (-raw) % self.tubelet_t


def _t(v) -> torch.Tensor:
    if isinstance(v, torch.Tensor):
        return v.detach().to(torch.float32).cpu()
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32))


def _attention(x, sd, pre, heads):
    """``_Attention.forward`` (model.py:34-40)."""
    b, t, d = x.shape
    qkv = F.linear(x, sd[pre + ".qkv.weight"], sd[pre + ".qkv.bias"])
    q, k, v = qkv.reshape(b, t, 3, heads, d // heads).permute(2, 0, 3, 1, 4)
    o = F.scaled_dot_product_attention(q, k, v)
    return F.linear(o.transpose(1, 2).reshape(b, t, d),
                    sd[pre + ".proj.weight"], sd[pre + ".proj.bias"])


def _ln(x, sd, pre):
    return F.layer_norm(x, (x.shape[-1],), sd[pre + ".weight"],
                        sd[pre + ".bias"], 1e-5)


def _block(x, sd, pre, heads):
    """``_Block.forward`` (model.py:56-64): spatial, temporal, MLP."""
    b, nt, ns, d = x.shape
    s = x.reshape(b * nt, ns, d)
    s = s + _attention(_ln(s, sd, pre + ".norm_s"), sd, pre + ".attn_s", heads)
    t = s.reshape(b, nt, ns, d).transpose(1, 2).reshape(b * ns, nt, d)
    t = t + _attention(_ln(t, sd, pre + ".norm_t"), sd, pre + ".attn_t", heads)
    x = t.reshape(b, ns, nt, d).transpose(1, 2)
    h = F.linear(_ln(x, sd, pre + ".norm_m"), sd[pre + ".mlp.0.weight"],
                 sd[pre + ".mlp.0.bias"])
    h = F.gelu(h)                                   # nn.GELU() default: erf
    return x + F.linear(h, sd[pre + ".mlp.2.weight"], sd[pre + ".mlp.2.bias"])


def forward(state: dict, arch: Arch, channels: int, stack, mask) -> torch.Tensor:
    """Reconstruct the last frame of ``stack``.

    stack: (b, f, c, h, w) float in [0, 1]; mask: (b, h, w) bool.
    Returns (b, c, h, w) float32.  Raises the reference's ValueErrors
    (model.py:93-98).
    """
    sd = {k: _t(v) for k, v in state.items()}
    stack = _t(stack)
    mask = torch.as_tensor(np.asarray(mask)).to(torch.bool) \
        if not isinstance(mask, torch.Tensor) else mask.cpu().to(torch.bool)
    b, f, c, h, w = stack.shape
    p, T, F_ = arch.patch, arch.tubelet_t, arch.stack_len
    if c != channels:                                            # model.py:93-94
        raise ValueError("expected %d channels, got %d" % (channels, c))
    if h % p or w % p:                                           # model.py:95-96
        raise ValueError("frame size must be a multiple of the patch edge")
    if f > F_:                                                   # model.py:97-98
        raise ValueError("stack longer than configured length")
    with torch.no_grad():
        if f < F_:                                               # model.py:99-101
            stack = torch.cat((stack[:, :1].expand(b, F_ - f, c, h, w), stack), 1)
        mf = mask.to(torch.float32)                              # model.py:102
        chan = torch.zeros(b, F_, 1, h, w)                       # model.py:105-107
        chan[:, -1, 0] = mf
        stack = stack.clone()                                    # model.py:108-109
        stack[:, -1] = stack[:, -1] * (1.0 - mf[:, None])
        x = torch.cat((stack, chan), 2).transpose(1, 2)          # model.py:110
        x = F.conv3d(x, sd["embed.weight"], sd["embed.bias"],    # model.py:111
                     stride=(T, p, p))
        _, d, nt, nh, nw = x.shape
        x = x.reshape(b, d, nt, nh * nw).permute(0, 2, 3, 1)     # model.py:112-113
        x = x + sd["time_pos"][:, None, :]                       # model.py:114
        for i in range(arch.layers):                             # model.py:115-116
            x = _block(x, sd, "blocks.%d" % i, arch.heads)
        x = _ln(x[:, -1], sd, "norm")                            # model.py:117
        out = F.linear(x, sd["head.weight"], sd["head.bias"])    # model.py:118
        out = out.reshape(b, nh, nw, T, p, p, c)[:, :, :, -1]    # model.py:119-121
        out = out.permute(0, 5, 1, 3, 2, 4).reshape(b, c, nh * p, nw * p)
        return torch.sigmoid(out)                                # model.py:122


def state_keys(layers: int) -> list[str]:
    """State-dict key order of ``MaskedVideoModel`` (registration order:
    own parameter ``time_pos`` first, then ``embed``, ``blocks``, ``norm``,
    ``head`` -- model.py:70-80)."""
    keys = ["time_pos", "embed.weight", "embed.bias"]
    for i in range(layers):
        pre = "blocks.%d." % i
        for sub in ("norm_s.weight", "norm_s.bias",
                    "attn_s.qkv.weight", "attn_s.qkv.bias",
                    "attn_s.proj.weight", "attn_s.proj.bias",
                    "norm_t.weight", "norm_t.bias",
                    "attn_t.qkv.weight", "attn_t.qkv.bias",
                    "attn_t.proj.weight", "attn_t.proj.bias",
                    "norm_m.weight", "norm_m.bias",
                    "mlp.0.weight", "mlp.0.bias", "mlp.2.weight", "mlp.2.bias"):
            keys.append(pre + sub)
    keys += ["norm.weight", "norm.bias", "head.weight", "head.bias"]
    return keys
