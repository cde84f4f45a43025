"""Protocol conformance driven by the reference's OWN client.

The reference's cross-package criterion 11 (pkg/nvrec/tests/
test_nvrec_acceptance.py:48-94) connects ``rgbdstream.recovery.RemoteBackend``
(recovery.py:290-348) to an echo ``RecoveryServer`` and checks the
handshake, the masked merge, and that a malformed request drops only its
connection.  Here the same unmodified client talks to OUR server.  The
reference package exists only in the build container, so the test skips
elsewhere (e.g. on the GPU box)."""

import os
import socket
import struct
import sys

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF_SRC),
                                reason="reference package not present (GPU box)")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF_SRC)
    try:
        from rgbdstream import recovery
        from rgbdstream.codec import CorruptionMask
        from rgbdstream.frames import Modality
    finally:
        sys.path.remove(REF_SRC)
    return recovery, CorruptionMask, Modality


def _depth_request(ref, seed=0):
    recovery, CorruptionMask, Modality = ref
    rng = np.random.default_rng(seed)
    plane = rng.integers(0, 200, (32, 32), dtype=np.uint8)
    refs = [rng.integers(0, 200, (32, 32), dtype=np.uint8) for _ in range(2)]
    grid = np.zeros((2, 2), dtype=bool)
    grid[0, 1] = True
    return recovery.RecoveryRequest(frame_id=7, modality=Modality.DEPTH, plane=plane,
                                    mask=CorruptionMask(grid), references=refs)


@pytest.mark.parametrize("max_connections", [1, 4])
def test_reference_client_against_our_echo_server(ref, max_connections):
    from paper_2604_27441_b200.server import RecoveryServer
    recovery, CorruptionMask, Modality = ref
    server = RecoveryServer(("127.0.0.1", 0), echo=True, max_connections=max_connections)
    server.start()
    try:
        client = recovery.RemoteBackend(server.addr, budget_ms=10_000.0)
        client.connect()
        assert client.supported == 0b11
        req = _depth_request(ref)
        resp = client.recover(req)
        assert not resp.fallback and not resp.timeout
        assert resp.plane.shape == req.plane.shape and (resp.plane == req.plane).all()
        rgb = recovery.RecoveryRequest(
            frame_id=9, modality=Modality.RGB,
            plane=np.random.default_rng(1).integers(0, 255, (32, 32, 3), dtype=np.uint8),
            mask=CorruptionMask(np.array([[True, False], [False, False]])),
            references=[np.zeros((32, 32, 3), dtype=np.uint8)])
        resp = client.recover(rgb)
        assert not resp.fallback and (resp.plane == rgb.plane).all()
        client.close()
        # malformed request: that connection is dropped, the server survives
        with socket.create_connection(server.addr, timeout=5.0) as sock:
            head = b""
            while len(head) < 4:
                head += sock.recv(4 - len(head))
            (n,) = struct.unpack("<I", head)
            while n:
                n -= len(sock.recv(n))
            sock.sendall(struct.pack("<I", 5) + b"\xff" * 5)
            assert sock.recv(1) == b""
        fresh = recovery.RemoteBackend(server.addr, budget_ms=10_000.0)
        assert not fresh.recover(_depth_request(ref, seed=2)).fallback
        fresh.close()
    finally:
        server.close()
