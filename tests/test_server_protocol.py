"""RecoveryServer wire protocol, echo mode (CPU-only): mirrors the
reference's pkg/nvrec/tests/test_nvrec_server.py echo/malformed cases and the
cross-package criterion 11 (test_nvrec_acceptance.py:48-94)."""

import socket
import struct

import numpy as np
import pytest

from paper_2604_27441_b200.data import MOD_DEPTH, MOD_RGB
from paper_2604_27441_b200.server import (MSG_HANDSHAKE, MSG_REQUEST, MSG_RESPONSE,
                                          PROTOCOL_VERSION, RecoveryServer)


@pytest.fixture
def echo_server():
    srv = RecoveryServer(("127.0.0.1", 0), echo=True)
    srv.start()
    yield srv
    srv.close()


def _recv_exact(sock, n):
    buf = b""
    while len(buf) < n:
        chunk = sock.recv(n - len(buf))
        if not chunk:
            break
        buf += chunk
    return buf


def _connect(srv):
    sock = socket.create_connection(srv.addr, timeout=5.0)
    (n,) = struct.unpack("<I", _recv_exact(sock, 4))
    return sock, _recv_exact(sock, n)


def _request(modality, frame_id, plane, grid, refs):
    h, w = plane.shape[:2]
    body = struct.pack("<BBIHHB", MSG_REQUEST, modality, frame_id, w, h, len(refs))
    body += np.packbits(grid.reshape(-1)).tobytes() + plane.tobytes()
    for r in refs:
        body += r.tobytes()
    return struct.pack("<I", len(body)) + body


def _roundtrip(sock, payload):
    sock.sendall(payload)
    head = _recv_exact(sock, 4)
    if len(head) < 4:
        return None
    (n,) = struct.unpack("<I", head)
    return _recv_exact(sock, n)


def test_handshake_bytes(echo_server):
    sock, body = _connect(echo_server)
    sock.close()
    assert body == bytes([MSG_HANDSHAKE, PROTOCOL_VERSION, 0b11])


def test_needs_checkpoint_or_echo():
    with pytest.raises(ValueError):
        RecoveryServer(("127.0.0.1", 0))


def test_echo_returns_plane(echo_server):
    sock, _ = _connect(echo_server)
    plane = np.arange(32 * 32, dtype=np.uint8).reshape(32, 32, 1)
    grid = np.zeros((2, 2), bool)
    grid[0, 1] = True
    body = _roundtrip(sock, _request(MOD_DEPTH, 9, plane, grid, [plane]))
    assert body[0] == MSG_RESPONSE and struct.unpack_from("<I", body, 1)[0] == 9
    assert body[5:] == plane.tobytes()
    rgb = np.random.default_rng(0).integers(0, 256, (16, 16, 3), dtype=np.uint8)
    body = _roundtrip(sock, _request(MOD_RGB, 1, rgb, np.ones((1, 1), bool), []))
    assert body[5:] == rgb.tobytes()
    for fid in (1, 2, 3):                     # sequential requests, one connection
        body = _roundtrip(sock, _request(MOD_DEPTH, fid, plane, grid, []))
        assert struct.unpack_from("<I", body, 1)[0] == fid
    sock.close()


@pytest.mark.parametrize("payload", [
    struct.pack("<I", 3) + b"\x01\x02",
    struct.pack("<I", 2) + b"\xff\x00",
    struct.pack("<I", 12) + struct.pack("<BBIHHB", MSG_REQUEST, 7, 0, 16, 16, 0),
])
def test_malformed_dropped_server_survives(echo_server, payload):
    sock, _ = _connect(echo_server)
    sock.sendall(payload)
    sock.close()
    sock2, body = _connect(echo_server)
    assert body[0] == MSG_HANDSHAKE
    plane = np.zeros((16, 16, 1), np.uint8)
    resp = _roundtrip(sock2, _request(MOD_DEPTH, 4, plane, np.zeros((1, 1), bool), []))
    sock2.close()
    assert resp is not None and resp[0] == MSG_RESPONSE


def test_wrong_length_dropped(echo_server):
    sock, _ = _connect(echo_server)
    plane = np.zeros((16, 16, 1), np.uint8)
    good = _request(MOD_DEPTH, 1, plane, np.zeros((1, 1), bool), [])
    sock.sendall(good[:-5] + struct.pack("<I", 0))
    sock.close()
    sock2, body = _connect(echo_server)
    sock2.close()
    assert body[0] == MSG_HANDSHAKE
