"""Precision experiment for the fp32-class tensor-core ("precise") path.

Re-runs the nvrec forward (oracle/nvrec_forward.py structure) with every
GEMM -- embed, qkv, attention QK^T and PV, proj, fc1, fc2 -- computed from
split 16-bit operands, a = hi + lo, as hi*hi + hi*lo + lo*hi with fp32
accumulation (what the tcgen05 kernels do), and reports the max-abs error
against the fp32 oracle on [0,1] outputs.  The head runs in fp32 (CUDA
cores) on the device too.

    python tools/precision_emul.py [--h 240 --w 320] [--fmt bf16|fp16]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import nvrec_forward as nf  # noqa: E402
from helpers import make_state, textured_u8, block_grid  # noqa: E402


def split(x, dt, terms=2):
    if dt is None:
        return [x]
    hi = x.to(dt).float()
    if terms == 1:
        return [hi]
    lo = (x - hi).to(dt).float()
    return [hi, lo]


def mm3(a, b, dt):
    """a @ b with split operands (hi.hi + hi.lo + lo.hi)."""
    if dt is None:
        return a @ b
    ah, al = split(a, dt)
    bh, bl = split(b, dt)
    return ah @ bh + ah @ bl + al @ bh


def linear(x, w, bias, dt):
    return mm3(x, w.t(), dt) + bias


def attention_sdpa(q, k, v, dt, dt_pv):
    s = mm3(q, k.transpose(-1, -2), dt) / np.sqrt(q.shape[-1])
    m = s.amax(-1, keepdim=True)
    p = torch.exp(s - m)
    l = p.sum(-1, keepdim=True)
    return mm3(p, v, dt_pv) / l


def forward(sd, arch, c, stack, mask, dt, dt_pv):
    b, f, _, h, w = stack.shape
    p, T, heads = arch.patch, arch.tubelet_t, arch.heads
    Fs = arch.stack_len
    if f < Fs:
        stack = torch.cat((stack[:, :1].expand(b, Fs - f, c, h, w), stack), 1)
    mf = mask.float()
    chan = torch.zeros(b, Fs, 1, h, w)
    chan[:, -1, 0] = mf
    stack = stack.clone()
    stack[:, -1] = stack[:, -1] * (1 - mf[:, None])
    x = torch.cat((stack, chan), 2).transpose(1, 2)           # (b, c+1, F, h, w)
    nt, nh, nw = Fs // T, h // p, w // p
    # patches: (b, nt, nh, nw, (c+1)*T*p*p) in conv weight order (ci, tt, py, px)
    xp = x.reshape(b, c + 1, nt, T, nh, p, nw, p).permute(0, 2, 4, 6, 1, 3, 5, 7)
    xp = xp.reshape(b, nt * nh * nw, -1)
    wemb = sd["embed.weight"].reshape(sd["embed.weight"].shape[0], -1)
    # pixels are exact in 16-bit (u8 * 255 scale): split only the weight
    pix = (xp * 255.0).round()
    if dt is None:
        acc = pix @ wemb.t()
    else:
        wh, wl = split(wemb, dt)
        acc = pix @ wh.t() + pix @ wl.t()
    x = acc / 255.0 + sd["embed.bias"]
    d = x.shape[-1]
    x = x.reshape(b, nt, nh * nw, d) + sd["time_pos"][:, None, :]

    def attn(xx, pre):
        bb, t, _ = xx.shape
        qkv = linear(xx, sd[pre + ".qkv.weight"], sd[pre + ".qkv.bias"], dt)
        q, k, v = qkv.reshape(bb, t, 3, heads, d // heads).permute(2, 0, 3, 1, 4)
        o = attention_sdpa(q, k, v, dt, dt_pv)
        return linear(o.transpose(1, 2).reshape(bb, t, d), sd[pre + ".proj.weight"],
                      sd[pre + ".proj.bias"], dt)

    def ln(xx, pre):
        return F.layer_norm(xx, (d,), sd[pre + ".weight"], sd[pre + ".bias"], 1e-5)

    for i in range(arch.layers):
        pre = "blocks.%d" % i
        ns = nh * nw
        s = x.reshape(b * nt, ns, d)
        s = s + attn(ln(s, pre + ".norm_s"), pre + ".attn_s")
        t = s.reshape(b, nt, ns, d).transpose(1, 2).reshape(b * ns, nt, d)
        t = t + attn(ln(t, pre + ".norm_t"), pre + ".attn_t")
        x = t.reshape(b, ns, nt, d).transpose(1, 2)
        hdn = F.gelu(linear(ln(x, pre + ".norm_m"), sd[pre + ".mlp.0.weight"],
                            sd[pre + ".mlp.0.bias"], dt))
        x = x + linear(hdn, sd[pre + ".mlp.2.weight"], sd[pre + ".mlp.2.bias"], dt)
    x = ln(x[:, -1], "norm")
    out = F.linear(x, sd["head.weight"], sd["head.bias"])
    out = out.reshape(b, nh, nw, T, p, p, c)[:, :, :, -1]
    out = out.permute(0, 5, 1, 3, 2, 4).reshape(b, c, nh * p, nw * p)
    return torch.sigmoid(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--h", type=int, default=240)
    ap.add_argument("--w", type=int, default=320)
    args = ap.parse_args()
    arch = nf.Arch()
    rng = np.random.default_rng(0)
    fmts = {"fp32": None, "bf16": torch.bfloat16, "fp16": torch.float16}
    for c in (3, 1):
        sd = {k: torch.from_numpy(v) for k, v in make_state(arch, c, seed=c).items()}
        fr = textured_u8(rng, 6, args.h, args.w, c)
        grid = block_grid(rng, args.h // 16, args.w // 16, 0.1)
        pix = np.repeat(np.repeat(grid, 16, 0), 16, 1)
        stack = torch.from_numpy(fr.astype(np.float32) / 255.0).permute(0, 3, 1, 2)[None]
        mask = torch.from_numpy(pix)[None]
        with torch.no_grad():
            ref = nf.forward(sd, arch, c, stack, mask)
            for name, (dt, dpv) in {"fp32-emul": (None, None),
                                    "bf16x3": (torch.bfloat16, torch.bfloat16),
                                    "fp16x3": (torch.float16, torch.float16),
                                    "bf16x3 qk + fp16x3 pv": (torch.bfloat16, torch.float16),
                                    }.items():
                out = forward(sd, arch, c, stack, mask, dt, dpv)
                err = (out - ref).abs()[:, :, pix].max().item() if False else \
                    (out - ref).abs().permute(0, 2, 3, 1)[0][torch.from_numpy(pix)].max().item()
                print("c=%d %dx%d %-24s max-abs %.3e  (%.2f LSB16)" %
                      (c, args.w, args.h, name, err, err * 65535))


if __name__ == "__main__":
    main()
