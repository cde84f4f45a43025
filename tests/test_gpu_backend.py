"""In-process backend (receiver callable) with the device-resident ring."""

from dataclasses import dataclass

import numpy as np
import pytest
import torch

from helpers import block_grid, make_state, textured_u8
from oracle import nvrec_forward, recover as oracle_recover

pytestmark = pytest.mark.gpu


@dataclass
class _Mask:
    grid: np.ndarray


@dataclass
class _Req:                      # field-compatible with rgbdstream RecoveryRequest
    frame_id: int
    modality: int
    plane: np.ndarray
    mask: _Mask
    references: list


def _ck(c, seed):
    from paper_2604_27441_b200 import Checkpoint, ModelConfig
    arch = nvrec_forward.Arch()
    st = make_state(arch, c, seed)
    return Checkpoint(ModelConfig(), c, {k: torch.from_numpy(v) for k, v in st.items()}), st


def test_backend_matches_oracle_and_uploads_one_plane_per_frame():
    from paper_2604_27441_b200.backend import B200Backend
    ck_d, st_d = _ck(1, 501)
    be = B200Backend(checkpoint_depth=ck_d)
    rng = np.random.default_rng(3)
    frames = textured_u8(rng, 12, 96, 128, 1)[..., 0]
    ring = [frames[i] for i in range(5)]
    arch = nvrec_forward.Arch()
    uploads = []
    for t in range(5, 12):
        grid = block_grid(rng, 6, 8, 0.3)
        grid[0, 0] = True
        plane = frames[t].copy()
        resp = be(_Req(t, 1, plane, _Mask(grid), list(ring)))
        want = oracle_recover.recover(st_d, arch, 1, plane[..., None], grid,
                                      [r[..., None] for r in ring])[..., 0]
        assert resp.plane.shape == plane.shape and not resp.fallback
        assert np.abs(resp.plane.astype(int) - want.astype(int)).max() <= 2
        uploads.append(be.caches[1].uploads)
        ring = ring[1:] + [resp.plane]          # receiver.py:268-269
    # first request uploads its 5 references; afterwards the ring is resident
    assert uploads[0] == 5 and uploads[-1] == 5


def test_backend_echo_rules():
    from paper_2604_27441_b200.backend import B200Backend
    ck_r, _ = _ck(3, 502)
    be = B200Backend(checkpoint_rgb=ck_r)
    plane = np.full((32, 32, 3), 9, np.uint8)
    g = np.ones((2, 2), bool)
    assert np.array_equal(be(_Req(1, 0, plane, _Mask(g), [])).plane, plane)       # no refs
    assert np.array_equal(be(_Req(1, 0, plane, _Mask(~g), [plane])).plane, plane)  # empty mask
    dep = np.full((32, 32), 4, np.uint8)
    assert np.array_equal(be(_Req(1, 1, dep, _Mask(g), [dep])).plane, dep)  # no depth model


def test_recovery_pipeline_matches_sequential_engine():
    """Double-buffered serving loop == per-request engine calls with the
    receiver's ring semantics (recovered plane joins the ring)."""
    from paper_2604_27441_b200.lossmask import PFrameShards
    from paper_2604_27441_b200.recovery import RecoveryEngine, RecoveryPipeline
    from tools.synth import p_frame_shards
    from oracle import lossmask as om
    ck, _ = _ck(3, 503)
    eng = RecoveryEngine(ck.build_model(), "fast")
    n, h, w, c, k = 2, 64, 96, 3, 5
    rng = np.random.default_rng(8)
    refs = [list(textured_u8(rng, k, h, w, c)) for _ in range(n)]
    init = torch.from_numpy(np.stack([np.stack(r) for r in refs])).cuda()
    pipe = RecoveryPipeline(eng, n, h, w, 1024, 2048, 64, init)
    handles, expected = [], []
    for step in range(4):
        planes = np.stack([textured_u8(rng, 1, h, w, c)[0] for _ in range(n)])
        jobs, outs = [], []
        for s in range(n):
            hdr, nd, recv, enc = p_frame_shards(rng, w, h, c, 64, lambda: rng.random() < 0.5,
                                                present_ratio=0.5)
            jobs.append(PFrameShards(hdr, nd, recv, 64, enc))
            grid = om.mask_from_shards(hdr, nd, {i for i in range(nd) if recv[i]}, 64, enc)
            o = eng.recover(planes[s], grid, refs[s])
            refs[s] = refs[s][1:] + [o]
            outs.append(o)
        expected.append(np.stack(outs))
        handles.append(pipe.submit(planes, jobs))
        if step >= 1:
            got = pipe.result(handles[step - 1])
            assert np.array_equal(got, expected[step - 1])
    assert np.array_equal(pipe.result(handles[-1]), expected[-1])


def test_receiver_pipeline_matches_reference_receiver_chain():
    """GPU receiver (decode -> mask -> recover -> in-place ring) == the
    reference receiver's chain restated with the oracle decode
    (codec.py:260-321, receiver.py:222-269) and per-request engine calls."""
    from tools import synth
    from paper_2604_27441_b200.receiver import ReceiverPipeline
    from paper_2604_27441_b200.recovery import RecoveryEngine
    from oracle import codec as oc
    ck, _ = _ck(3, 504)
    eng = RecoveryEngine(ck.build_model(), "fast")
    n, h, w, c, k, L = 2, 64, 96, 3, 5, 256
    rng = np.random.default_rng(9)
    clips = [synth.talking_clip(12, w, h, c, seed=40 + s, motion_fraction=0.3) for s in range(n)]
    # the sender encodes against its own clean reconstruction
    enc, refs, disp = [], [], []
    for s in range(n):
        hi, pi = synth.encode_i(clips[s][0])
        rec, _ = oc.decode(hi, pi)
        seq = []
        for f in clips[s][1:]:
            hp, pp = synth.encode_p(f, rec)
            rec, _ = oc.decode(hp, pp, rec)
            seq.append((hp, pp))
        enc.append(seq)
        refs.append([clips[s][0]] * k)
        disp.append(clips[s][0])
    init = torch.from_numpy(np.stack([np.stack(r) for r in refs])).cuda()
    pipe = ReceiverPipeline(eng, n, h, w, init, 4096, 1 << 16, 64)
    for step in range(6):
        frames, expected = [], []
        for s in range(n):
            hp, pp = enc[s][step]
            nd = synth.n_data_shards(len(pp), L)
            recv = np.ones(nd, bool)
            recv[1:] = rng.random(nd - 1) >= 0.3
            body = synth.receiver_body(pp, L, recv)
            frames.append((hp, body, recv, L))
            shards = {i: pp[(i - 1) * L:i * L] for i in range(1, nd) if recv[i]}
            b2, zf = oc.finalize_p_body(nd, shards, L, len(pp))
            assert b2 == body
            plane, grid = oc.decode(hp, b2, disp[s], zf)
            out = eng.recover(plane, grid, refs[s]) if grid.any() else plane
            refs[s] = refs[s][1:] + [out]
            disp[s] = out
            expected.append(out)
        hnd = pipe.submit(frames)
        got, st = pipe.result(hnd)
        assert not st.any()
        assert np.array_equal(got, np.stack(expected))


def test_concurrent_pinned_server_matches_engine():
    """GPU front end (8f rank 2): several connections served concurrently
    through pinned buffers return exactly what the per-request engine does,
    including refs > k and the echo rules."""
    import socket
    import struct
    import threading
    from paper_2604_27441_b200.recovery import RecoveryEngine
    from paper_2604_27441_b200.server import MSG_REQUEST, RecoveryServer
    ck_r, _ = _ck(3, 505)
    ck_d, _ = _ck(1, 506)
    srv = RecoveryServer(("127.0.0.1", 0), checkpoint_rgb=ck_r, checkpoint_depth=ck_d,
                         max_connections=4)
    srv.start()
    engines = {0: RecoveryEngine(ck_r.build_model(), "fast"),
               1: RecoveryEngine(ck_d.build_model(), "fast")}
    errors = []

    def client(cid):
        try:
            rng = np.random.default_rng(cid)
            sock = socket.create_connection(srv.addr, timeout=30.0)
            (n,) = struct.unpack("<I", sock.recv(4))
            sock.recv(n)
            for it in range(4):
                mod = (cid + it) % 2
                c = 3 if mod == 0 else 1
                h, w, k = 48, 64, [0, 2, 5, 7][it]
                plane = textured_u8(rng, 1, h, w, c)[0]
                refs = list(textured_u8(rng, k, h, w, c)) if k else []
                grid = rng.random((h // 16, w // 16)) < 0.4
                body = struct.pack("<BBIHHB", MSG_REQUEST, mod, it, w, h, k)
                body += np.packbits(grid.reshape(-1)).tobytes() + plane.tobytes()
                body += b"".join(r.tobytes() for r in refs)
                sock.sendall(struct.pack("<I", len(body)) + body)
                buf = b""
                while len(buf) < 4:
                    buf += sock.recv(4 - len(buf))
                (n,) = struct.unpack("<I", buf)
                resp = b""
                while len(resp) < n:
                    resp += sock.recv(n - len(resp))
                got = np.frombuffer(resp[5:], np.uint8).reshape(h, w, c)
                want = engines[mod].recover(plane, grid, refs) if refs and grid.any() else plane
                if not np.array_equal(got, want.reshape(h, w, c)):
                    errors.append((cid, it))
            sock.close()
        except Exception as exc:          # noqa: BLE001
            errors.append((cid, repr(exc)))

    threads = [threading.Thread(target=client, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(120)
    srv.close()
    assert not errors, errors
