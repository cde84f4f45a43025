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
  tests/golden/ssim_golden.npz     rgbdstream.metrics.ssim values
                                   (reference metrics.py:41-72)

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


def gen_codec():
    """Reference frame decode (codec.decode, codec.py:260-321) driven three
    ways: (1) the receiver's P-frame finalisation with Bernoulli body-shard
    loss (receiver.py:211-274; the plane handed to the recovery backend),
    (2) the receiver's I-frame finalisation with RS erasures
    (receiver.py:180-209 -> fec.rs_reconstruct -> codec.decode_bytes) and
    (3) direct codec.decode calls on crafted / malformed payloads.  Stores
    the encoded bytes and reference planes (inputs) and sha256 digests of the
    decoded planes + the grids (outputs)."""
    import hashlib
    import struct as st
    from rgbdstream import codec
    from rgbdstream.codec import CodecConfig, EncodedFrame
    from rgbdstream.fec import ProtectionPolicy, plan_protection, rs_encode
    from rgbdstream.frames import FrameKind, GoPSpec, Modality
    from rgbdstream.packet import packetize
    from rgbdstream.receiver import FrameAssembly, Receiver
    from rgbdstream.recovery import RecoveryResponse
    from rgbdstream.synthetic import talking_motion_clip

    cfg = CodecConfig()
    policy = ProtectionPolicy()
    rng = np.random.default_rng(4242)
    blobs, refs = [], []           # byte strings / reference planes (deduplicated by index)
    trials = []

    def blob(b):
        blobs.append(np.frombuffer(bytes(b), np.uint8))
        return len(blobs) - 1

    def refplane(a):
        refs.append(np.ascontiguousarray(a))
        return len(refs) - 1

    def dg(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

    seen = {}

    def backend(req):
        seen["plane"] = req.plane.copy()
        seen["grid"] = req.mask.grid.copy()
        return RecoveryResponse(req.plane.copy(), 0.0)

    for (w, h, nf) in ((64, 64, 5), (128, 96, 5), (320, 240, 5), (640, 480, 2)):
        clip = talking_motion_clip(nf, w, h, seed=w * 7 + h)
        for mod in (Modality.RGB, Modality.DEPTH):
            L = 1024 if mod == Modality.RGB else 512
            planes = [f.rgb if mod == Modality.RGB else f.depth for f in clip]
            ienc = codec.encode_i(planes[0], cfg, frame_id=0, modality=mod)
            idata = ienc.to_bytes()
            ib = blob(idata)
            plan = plan_protection(FrameKind.I, len(idata), policy, L)
            clean0, _ = codec.decode(ienc)
            # I-frame trials through the receiver (RS reconstruct + decode_bytes)
            pk = packetize(ienc, plan, policy)
            nt = plan.n + plan.r
            pats = [np.ones(nt, bool)]
            for p in (0.1, 0.3):
                pats.append(rng.random(nt) >= p)
            worst = np.ones(nt, bool)
            worst[rng.choice(plan.n, min(plan.r, plan.n), replace=False)] = False
            pats.append(worst)
            over = np.ones(nt, bool)
            over[rng.choice(nt, plan.r + 1, replace=False)] = False
            pats.append(over)
            for pres in pats:
                rec = Receiver(GoPSpec(), cfg)
                asm = FrameAssembly(0, mod, FrameKind.I, plan.n, plan.r, len(idata),
                                    first_packet_ts=0.0)
                for q in pk:
                    if pres[q.shard_index]:
                        asm.shards[q.shard_index] = q.payload
                out = rec._finalize_i(0, mod, 0, asm)
                ok = out.plane is not None
                trials.append(dict(kind="iframe", data=ib, n=plan.n, r=plan.r, L=plan.shard_len,
                                   present=pres.astype(np.uint8), err="" if ok else "lost",
                                   digest=dg(out.plane) if ok else "",
                                   grid=(out.mask.grid.reshape(-1) if ok else np.zeros(0, bool)),
                                   parity_digest=dg(np.frombuffer(b"".join(
                                       rs_encode(idata, plan.n, plan.r, plan.shard_len)
                                       .shards[plan.n:]), np.uint8))))
            ref = clean0
            for fi in range(1, nf):
                enc = codec.encode_p(planes[fi], ref, cfg, frame_id=fi, modality=mod)
                clean, _ = codec.decode(enc, ref)
                hb, pb, rp = blob(enc.header), blob(enc.payload), refplane(ref)
                pplan = plan_protection(FrameKind.P, enc.encoded_len, policy, L,
                                        header_len=len(enc.header))
                pkts = packetize(enc, pplan, policy)
                for p in (0.0, 0.05, 0.2, 0.5):
                    rec = Receiver(GoPSpec(), cfg, backend=backend)
                    rec.refs[mod] = ref
                    asm = FrameAssembly(fi, mod, FrameKind.P, pplan.n, pplan.r,
                                        enc.encoded_len, first_packet_ts=0.0)
                    for q in pkts:
                        if q.shard_index == 0 or rng.random() >= p:
                            asm.shards.setdefault(q.shard_index, q.payload)
                    seen.clear()
                    out = rec._finalize_p(fi, mod, 0, asm)
                    plane = seen.get("plane", out.plane)
                    grid = seen.get("grid", out.mask.grid if out.mask is not None else None)
                    received = np.array([i in asm.shards for i in range(pplan.n)], np.uint8)
                    trials.append(dict(kind="pframe", header=hb, payload=pb, ref=rp,
                                       n=pplan.n, L=L, encoded_len=enc.encoded_len,
                                       present=received, err="", digest=dg(plane),
                                       grid=np.asarray(grid, bool).reshape(-1)))
                ref = clean

    # crafted / malformed payloads through codec.decode directly
    def direct(name, header, payload, ref, ranges=()):
        try:
            plane, m = codec.decode(EncodedFrame(0, 0, FrameKind(header[0]) if header[0] < 2
                                                 else FrameKind.P, Modality.RGB,
                                                 bytes(header), bytes(payload)),
                                    ref, list(ranges))
            err, d, g = "", dg(plane), m.grid.reshape(-1)
        except (codec.UndecodableError, ValueError) as e:
            err, d, g = str(e) or type(e).__name__, "", np.zeros(0, bool)
        trials.append(dict(kind="direct", name=name, header=blob(header), payload=blob(payload),
                           ref=-1 if ref is None else refplane(ref),
                           ranges=np.asarray(ranges, np.int64).reshape(-1, 2), err=err,
                           digest=d, grid=g))

    clip = talking_motion_clip(3, 128, 96, seed=9)
    ref, _ = codec.decode(codec.encode_i(clip[0].rgb, cfg))
    enc = codec.encode_p(clip[1].rgb, ref, cfg)
    H, P = bytearray(enc.header), enc.payload
    npres = st.unpack_from("<H", H, 12)[0]
    bml = (st.unpack_from("<H", H, 2)[0] // 16) * (st.unpack_from("<H", H, 4)[0] // 16)
    bml = (bml + 7) // 8
    ooff = 14 + bml
    plen = len(P)
    direct("clean", H, P, ref)
    direct("tail_half", H, P[:plen // 2], ref)
    direct("tail_empty", H, b"", ref)
    direct("explicit_ranges", H, P, ref, [(0, 3), (plen - 1, plen), (7, 7)])
    direct("inverted_range", H, P, ref, [(9, 2)])
    direct("p_without_ref", H, P, None)
    if npres >= 3:
        # shift block 1's start by one byte: records straddle ranges
        h2 = bytearray(H)
        o1 = st.unpack_from("<I", h2, ooff + 4)[0]
        st.pack_into("<I", h2, ooff + 4, o1 + 1)
        direct("straddle_shift1", h2, P, ref)
        h3 = bytearray(H)
        st.pack_into("<I", h3, ooff + 4, o1 + 3)           # whole record moves blocks
        direct("shift_one_record", h3, P, ref)
        h4 = bytearray(H)
        o2 = st.unpack_from("<I", h4, ooff + 8)[0]
        st.pack_into("<I", h4, ooff + 4, o2 + 3)          # block 1 range inverted
        direct("inverted_offsets", h4, P, ref)
        h5 = bytearray(H)
        st.pack_into("<I", h5, ooff + 4, o1 + 2)
        direct("straddle_shift2", h5, P, ref, [(0, 1)])
        direct("not_whole_records", h2, P, ref, [(0, 1)])
    direct("bad_count", H, P[:-3] + b"\x01\x00\x00", ref)
    direct("payload_longer", H, P + b"\x05\x02\x00" * 4, ref)
    # one present block, crafted extreme values: int16 wrap of unzigzag*quant+ref
    for quant, vals in ((255, [65535, 65534, 1, 2, 40000, 0]), (4, [65535, 32768, 32769, 7]),
                        (1, [510, 511, 3, 4])):
        for kind in (0, 1):
            c, w_, h_ = 3, 32, 16
            bs = 16 * 16 * c
            recs = []
            left, k = bs, 0
            while left:
                run = min(left, 97 + 31 * k)
                recs.append((run, vals[k % len(vals)]))
                left -= run
                k += 1
            recs.insert(1, (0, 12345))                       # zero-run record
            pay = b"".join(st.pack("<BH", r_, v_) for r_, v_ in recs)
            present = np.array([False, True])
            hdr = (st.pack("<BBHHBBIH", kind, c, w_, h_, 16, quant, len(pay), 1)
                   + np.packbits(present).tobytes() + st.pack("<I", 0))
            base = np.random.default_rng(quant + kind).integers(0, 256, (h_, w_, c)).astype(np.uint8)
            direct("crafted_q%d_k%d" % (quant, kind), hdr, pay, base if kind == 1 else None)
    bad = bytearray(H)
    bad[0] = 3
    direct("bad_kind", bad, P, ref)
    # I-frame decode through decode_bytes with a header-overlapping range
    idata = codec.encode_i(clip[2].rgb, cfg).to_bytes()
    try:
        codec.decode_bytes(idata, zero_fill_ranges=[(3, 40)])
        herr = ""
    except codec.UndecodableError as e:
        herr = str(e)
    trials.append(dict(kind="bytes", data=blob(idata), ranges=np.array([[3, 40]], np.int64),
                       err=herr, digest="", grid=np.zeros(0, bool)))

    # pack: blobs and refs ragged, trials as parallel arrays / json
    import json
    meta = []
    for t in trials:
        m = {k: (v if not isinstance(v, np.ndarray) else None) for k, v in t.items()}
        for k in ("present", "grid", "ranges"):
            m.pop(k, None)
        meta.append(m)
    def ragged(arrs, dtype):
        flat = np.concatenate([np.asarray(a, dtype).reshape(-1) for a in arrs]) if arrs else \
            np.zeros(0, dtype)
        off = np.cumsum([0] + [np.asarray(a).size for a in arrs]).astype(np.int64)
        return flat, off
    bflat, boff = ragged(blobs, np.uint8)
    rflat, roff = ragged(refs, np.uint8)
    rshape = np.array([list(r.shape) + [1] * (3 - r.ndim) for r in refs], np.int64)
    rnd = np.array([r.ndim for r in refs], np.int64)
    pres = ragged([t.get("present", np.zeros(0)) for t in trials], np.uint8)
    grids = ragged([t.get("grid", np.zeros(0)) for t in trials], np.uint8)
    rng_ = ragged([t.get("ranges", np.zeros((0, 2))) for t in trials], np.int64)
    np.savez_compressed(os.path.join(HERE, "codec_golden.npz"), blobs=bflat, blobs_off=boff,
                        refs=rflat, refs_off=roff, refs_shape=rshape, refs_ndim=rnd,
                        present=pres[0], present_off=pres[1], grid=grids[0], grid_off=grids[1],
                        ranges=rng_[0], ranges_off=rng_[1],
                        meta=np.array(json.dumps(meta)))
    print("codec trials", len(trials), "blobs", len(blobs), "bytes", bflat.size,
          "refs", len(refs), "errors", sum(1 for t in trials if t["err"]))


def gen_ssim():
    """rgbdstream.metrics.ssim (metrics.py:41-72) on seeded plane pairs."""
    from golden_cases import SSIM_CASES, ssim_case
    from rgbdstream.metrics import ssim
    out = {}
    for name in SSIM_CASES:
        a, b = ssim_case(name)
        out[name] = np.array(ssim(a, b), np.float64)
        out[name + "__digest"] = np.array(digest(a, b))
        print("ssim", name, a.shape, float(out[name]))
    np.savez_compressed(os.path.join(HERE, "ssim_golden.npz"), **out)


if __name__ == "__main__":
    torch.set_num_threads(8)
    import sys as _sys
    which = _sys.argv[1:] or ["lossmask", "model", "recover", "baseline", "codec", "ssim"]
    for w in which:
        globals()["gen_" + w]()
