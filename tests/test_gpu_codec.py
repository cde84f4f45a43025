"""GPU frame decode (nvrec_decode) and RS reconstruction (nvrec_rs_*):
bit-exact against the golden outputs of the UNMODIFIED reference
(tests/golden/codec_golden.npz) and against the oracle on synthetic
720p / 1080p streams."""

import numpy as np
import pytest
import torch

from codec_cases import blob, i_shards, p_body, ref_plane, sha, trials
from oracle import codec as oc

pytestmark = pytest.mark.gpu


def _codec():
    from paper_2604_27441_b200 import codec
    return codec


def _dev(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.reshape(a.shape[0], a.shape[1], -1)).cuda()


def test_pframe_receiver_trials_batched():
    cd = _codec()
    ts = list(trials("pframe"))
    batch = cd.DecodeBatch(len(ts), 4096, 1 << 20, 1200, max_shards=300)
    items, outs = [], []
    for t in ts:
        header, shards, body_len = p_body(t)
        body, _ = oc.finalize_p_body(t["n"], shards, t["L"], body_len)
        ref = _dev(ref_plane(t["ref"]))
        out = torch.empty_like(ref)
        outs.append(out)
        items.append(cd.DecodeItem(header, body, out, ref, n_data=t["n"],
                                   received=t["present"], shard_len=t["L"], body_len=body_len))
    batch.stage(items)
    batch.launch()
    grids = batch.grids()
    for t, out, g in zip(ts, outs, grids):
        plane = out.cpu().numpy()
        plane = plane[:, :, 0] if plane.shape[2] == 1 else plane
        assert sha(plane) == t["digest"]
        assert np.array_equal(g.reshape(-1), t["grid"])
    # the wire bits are np.packbits of the grid (recovery.py:221)
    w = batch.wire[:len(ts)].cpu().numpy()
    for j, t in enumerate(ts):
        nb = (t["grid"].size + 7) // 8
        assert np.array_equal(w[j, :nb], np.packbits(t["grid"]))


def test_pframe_in_place_decode_into_reference_slot():
    cd = _codec()
    t = next(t for t in trials("pframe") if t["grid"].any())
    header, shards, body_len = p_body(t)
    body, _ = oc.finalize_p_body(t["n"], shards, t["L"], body_len)
    slot = _dev(ref_plane(t["ref"]))
    batch = cd.DecodeBatch(1, 4096, 1 << 20, 1200, max_shards=300)
    batch.stage([cd.DecodeItem(header, body, slot, slot, n_data=t["n"], received=t["present"],
                               shard_len=t["L"], body_len=body_len)])
    batch.launch()
    batch.check()
    p = slot.cpu().numpy()
    assert sha(p[:, :, 0] if p.shape[2] == 1 else p) == t["digest"]


def test_iframe_rs_and_decode():
    cd = _codec()
    n_ok = 0
    for t in trials("iframe"):
        data, shards = i_shards(t)

        class S:
            pass
        s = S()
        s.n, s.r, s.shard_len, s.data_len = t["n"], t["r"], t["L"], len(data)
        s.shards, s.present = shards, [x is not None for x in shards]
        if t["err"]:
            with pytest.raises(cd.UnrecoverableError):
                cd.rs_reconstruct(s)
            continue
        got = cd.rs_reconstruct(s)
        assert got == data
        plane, mask = cd.decode_bytes(got)
        assert sha(plane) == t["digest"]
        assert np.array_equal(mask.grid.reshape(-1), t["grid"])
        n_ok += 1
    assert n_ok >= 10


def test_direct_cases_match_reference():
    cd = _codec()
    for t in trials("direct"):
        hdr, pay, ref = blob(t["header"]), blob(t["payload"]), ref_plane(t["ref"])
        if t["err"]:
            with pytest.raises(ValueError) as ei:
                cd.decode((hdr, pay), ref, t["ranges"])
            assert str(ei.value) == t["err"], t["name"]
            continue
        plane, mask = cd.decode((hdr, pay), ref, t["ranges"])
        assert sha(plane) == t["digest"], t["name"]
        assert np.array_equal(mask.grid.reshape(-1), t["grid"]), t["name"]
    for t in trials("bytes"):
        with pytest.raises(ValueError, match=t["err"]):
            cd.decode_bytes(blob(t["data"]), zero_fill_ranges=t["ranges"])


def _scene(rng, h, w, c):
    """Coarse textured plane + a moving re-textured patch (talking-motion-like)."""
    cell = 8
    base = rng.integers(0, 256, (h // cell + 1, w // cell + 1, c), dtype=np.uint8)
    a = np.repeat(np.repeat(base, cell, 0), cell, 1)[:h, :w]
    return a if c > 1 else a[:, :, 0]


@pytest.mark.parametrize("h,w,c,L,p", [(720, 1280, 3, 1024, 0.05), (720, 1280, 1, 512, 0.2),
                                       (1088, 1920, 3, 1024, 0.2), (480, 640, 1, 512, 0.5)])
def test_large_stream_vs_oracle(h, w, c, L, p):
    from tools import synth
    cd = _codec()
    rng = np.random.default_rng(h + c)
    f0 = _scene(rng, h, w, c)
    hdr_i, pay_i = synth.encode_i(f0)
    ref_o, _ = oc.decode(hdr_i, pay_i)
    plane_g, _ = cd.decode((hdr_i, pay_i))
    assert np.array_equal(plane_g, ref_o)
    f1 = f0.copy()
    ph, pw = h // 4, w // 4
    f1[h // 3:h // 3 + ph, w // 3:w // 3 + pw] = _scene(rng, ph, pw, c)
    f1 = np.clip(f1.astype(int) + rng.integers(-9, 10, f1.shape), 0, 255).astype(np.uint8)
    hdr, pay = synth.encode_p(f1, ref_o)
    nd = synth.n_data_shards(len(pay), L)
    received = np.ones(nd, bool)
    received[1:] = rng.random(nd - 1) >= p
    shards = {i: pay[(i - 1) * L:i * L] for i in range(1, nd) if received[i]}
    body, zf = oc.finalize_p_body(nd, shards, L, len(pay))
    want_plane, want_grid = oc.decode(hdr, body, ref_o, zf)
    ref_d = _dev(ref_o)
    out = torch.empty_like(ref_d)
    batch = cd.DecodeBatch(1, len(hdr), len(body), (h // 16) * (w // 16), max_shards=nd)
    batch.stage([cd.DecodeItem(hdr, body, out, ref_d, n_data=nd, received=received,
                               shard_len=L, body_len=len(pay))])
    batch.launch()
    g = batch.grids()[0]
    got = out.cpu().numpy()
    assert np.array_equal(g, want_grid)
    assert np.array_equal(got[:, :, 0] if c == 1 else got, want_plane)
    assert want_grid.any()


@pytest.mark.parametrize("n,r,L", [(170, 85, 16384), (200, 55, 1001), (5, 3, 64), (1, 1, 4)])
def test_rs_reconstruct_vs_oracle(n, r, L):
    from tools import synth
    cd = _codec()
    rng = np.random.default_rng(n * 7 + r)
    data = rng.integers(0, 256, n * L - 3, dtype=np.uint8).tobytes()
    full = [data[i * L:(i + 1) * L].ljust(L, b"\0") for i in range(n)] + \
        synth.rs_parity(data, n, r, L)
    lost = rng.choice(n + r, r, replace=False)
    shards = [None if i in lost else x for i, x in enumerate(full)]

    class S:
        pass
    s = S()
    s.n, s.r, s.shard_len, s.data_len = n, r, L, len(data)
    s.shards, s.present = shards, [x is not None for x in shards]
    assert cd.rs_reconstruct(s) == oc.rs_reconstruct(n, r, L, len(data), shards) == data
