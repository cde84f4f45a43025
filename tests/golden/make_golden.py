"""Generate the golden fixtures by running the UNMODIFIED reference.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/model_golden.npz    MaskedVideoModel.forward outputs
                                   (reference pkg/nvrec/src/nvrec/model.py:82-122)
  tests/golden/recover_golden.npz  RecoveryServer._recover outputs
                                   (reference pkg/nvrec/src/nvrec/server.py:181-196)
  tests/golden/lossmask_golden.npz receiver+codec corruption masks
                                   (reference receiver.py:211-274, codec.py:260-321)

Inputs are NOT stored: they are rebuilt from seeds by
``tests/golden_cases.py`` (and digests are stored to catch drift).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
TESTS = os.path.dirname(HERE)
sys.path.insert(0, TESTS)
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "nvrec", "src"))

from golden_cases import (BASELINE_CASES, MODEL_CASES, RECOVER_CASES,  # noqa: E402
                          baseline_case, model_case, recover_case)
from helpers import digest  # noqa: E402

from nvrec.config import ModelConfig  # noqa: E402
from nvrec.model import MaskedVideoModel  # noqa: E402
from nvrec.server import RecoveryServer  # noqa: E402
from nvrec.train import Checkpoint  # noqa: E402


def _ref_model(arch, c, state):
    cfg = ModelConfig(k=arch.k, tubelet_t=arch.tubelet_t, patch=arch.patch,
                      dim=arch.dim, layers=arch.layers, heads=arch.heads)
    m = MaskedVideoModel(cfg, c)
    m.load_state_dict({k: torch.from_numpy(v) for k, v in state.items()})
    return m.eval(), cfg


def gen_model():
    out = {}
    for name in MODEL_CASES:
        arch, c, state, stack, mask = model_case(name)
        m, _ = _ref_model(arch, c, state)
        with torch.no_grad():
            y = m(torch.from_numpy(stack), torch.from_numpy(mask)).numpy()
        out[name] = y.astype(np.float32)
        out[name + "__digest"] = np.array(digest(stack, mask, *state.values()))
        print("model", name, y.shape, float(y.min()), float(y.max()))
    np.savez_compressed(os.path.join(HERE, "model_golden.npz"), **out)


def gen_recover():
    out = {}
    for name in RECOVER_CASES:
        arch, c, state, plane, grid, refs = recover_case(name)
        _, cfg = _ref_model(arch, c, state)
        ck = Checkpoint(config=cfg, channels=c,
                        state={k: torch.from_numpy(v) for k, v in state.items()})
        kw = {"checkpoint_rgb": ck} if c == 3 else {"checkpoint_depth": ck}
        srv = RecoveryServer(("127.0.0.1", 0), **kw)
        try:
            mod = 0 if c == 3 else 1
            got = srv._recover(mod, plane, grid, refs)
        finally:
            srv.listener.close()
        out[name] = np.ascontiguousarray(got)
        out[name + "__digest"] = np.array(digest(plane, grid, *refs, *state.values()))
        print("recover", name, got.shape, int((got != plane).sum()))
    np.savez_compressed(os.path.join(HERE, "recover_golden.npz"), **out)


def gen_lossmask():
    """Drive the reference receiver's P-frame finalisation on real encoded
    frames with Bernoulli body-shard loss and record the mask it hands to
    the recovery backend (receiver.py:260-264)."""
    from rgbdstream import codec
    from rgbdstream.codec import CodecConfig
    from rgbdstream.fec import ProtectionPolicy, plan_protection
    from rgbdstream.frames import FrameKind, GoPSpec, Modality
    from rgbdstream.packet import packetize
    from rgbdstream.receiver import FrameAssembly, Receiver
    from rgbdstream.recovery import RecoveryResponse
    from rgbdstream.synthetic import talking_motion_clip

    cfg = CodecConfig()
    policy = ProtectionPolicy()
    rows = []            # per-trial dicts
    seen = {}

    def backend(req):
        seen["mask"] = req.mask.grid.copy()
        return RecoveryResponse(req.plane.copy(), 0.0)

    trial_rng = np.random.default_rng(2604)
    sizes = [(64, 64), (128, 96), (320, 240)]
    for (w, h) in sizes:
        clip = talking_motion_clip(7, w, h, seed=w + h)
        for mod in (Modality.RGB, Modality.DEPTH):
            L = 1024 if mod == Modality.RGB else 512
            planes = [f.rgb if mod == Modality.RGB else f.depth for f in clip]
            ienc = codec.encode_i(planes[0], cfg, frame_id=0, modality=mod)
            ref, _ = codec.decode(ienc)
            for fi in range(1, len(planes)):
                enc = codec.encode_p(planes[fi], ref, cfg, frame_id=fi,
                                     modality=mod)
                clean, _ = codec.decode(enc, ref)
                plan = plan_protection(FrameKind.P, enc.encoded_len, policy, L,
                                       header_len=len(enc.header))
                pkts = packetize(enc, plan, policy)
                for p in (0.0, 0.05, 0.1, 0.2, 0.5, 1.0):
                    rec = Receiver(GoPSpec(), cfg, backend=backend)
                    rec.refs[mod] = ref
                    asm = FrameAssembly(fi, mod, FrameKind.P, plan.n, plan.r,
                                        enc.encoded_len, first_packet_ts=0.0)
                    for pk in pkts:
                        if pk.shard_index == 0 or trial_rng.random() >= p:
                            asm.shards.setdefault(pk.shard_index, pk.payload)
                    seen.clear()
                    outc = rec._finalize_p(fi, mod, 0, asm)
                    grid = outc.mask.grid if outc.mask is not None else None
                    if "mask" in seen:
                        assert np.array_equal(seen["mask"], grid)
                    received = np.array([i in asm.shards for i in range(plan.n)])
                    rows.append(dict(header=np.frombuffer(enc.header, np.uint8),
                                     n_data=plan.n, shard_len=L,
                                     encoded_len=enc.encoded_len,
                                     received=received,
                                     grid=np.asarray(grid, bool).reshape(-1),
                                     gh=h // 16, gw=w // 16))
                ref = clean
    # codec-level tail rule (codec.py:274-278): truncated payload, no ranges,
    # plus explicit single ranges and an empty range
    extra = []
    clip = talking_motion_clip(3, 64, 64, seed=5)
    ienc = codec.encode_i(clip[0].rgb, cfg)
    ref, _ = codec.decode(ienc)
    enc = codec.encode_p(clip[1].rgb, ref, cfg, frame_id=1)
    plen = len(enc.payload)
    for cut, zr in ((plen // 2, []), (plen, [(0, 3)]), (plen, [(5, 5)]),
                    (plen, [(plen - 1, plen)]), (0, []), (plen, [(3, 2)])):
        e2 = codec.EncodedFrame(1, 0, FrameKind.P, Modality.RGB, enc.header,
                                enc.payload[:cut])
        try:
            _, m = codec.decode(e2, ref, zr)
            g = m.grid.reshape(-1)
        except codec.UndecodableError:
            continue
        extra.append(dict(header=np.frombuffer(enc.header, np.uint8),
                          received_len=cut,
                          ranges=np.array(zr, np.int64).reshape(-1, 2),
                          grid=g.astype(bool)))

    def pack(rows, keys_var, keys_fix):
        d = {}
        for k in keys_var:
            arrs = [np.asarray(r[k]) for r in rows]
            d[k] = np.concatenate([a.reshape(-1) if k != "ranges" else a
                                   for a in arrs]) if arrs else np.zeros(0)
            d[k + "_off"] = np.cumsum([0] + [len(a) for a in arrs]).astype(np.int64)
        for k in keys_fix:
            d[k] = np.array([r[k] for r in rows], np.int64)
        return d

    d = pack(rows, ["header", "received", "grid"],
             ["n_data", "shard_len", "encoded_len", "gh", "gw"])
    e = pack(extra, ["header", "ranges", "grid"], ["received_len"])
    np.savez_compressed(os.path.join(HERE, "lossmask_golden.npz"),
                        **d, **{"x_" + k: v for k, v in e.items()})
    n_flag = int(d["grid"].sum())
    print("lossmask trials", len(rows), "flagged blocks", n_flag,
          "codec cases", len(extra))


def gen_baseline():
    """Reference timeout/fault fallback (rgbdstream/recovery.py:128-196)."""
    from rgbdstream.codec import CorruptionMask
    from rgbdstream.frames import Modality
    from rgbdstream.recovery import RecoveryRequest, recover_baseline
    out = {}
    for name in BASELINE_CASES:
        c, plane, grid, refs = baseline_case(name)
        mod = Modality.RGB if c == 3 else Modality.DEPTH
        resp = recover_baseline(RecoveryRequest(1, mod, plane, CorruptionMask(grid.copy()),
                                                refs))
        out[name] = resp.plane
        out[name + "__digest"] = np.array(digest(plane, grid, *refs))
        print("baseline", name, resp.plane.shape, int((resp.plane != plane).sum()))
    np.savez_compressed(os.path.join(HERE, "baseline_golden.npz"), **out)


if __name__ == "__main__":
    torch.set_num_threads(8)
    import sys as _sys
    which = _sys.argv[1:] or ["lossmask", "model", "recover", "baseline"]
    for w in which:
        globals()["gen_" + w]()
