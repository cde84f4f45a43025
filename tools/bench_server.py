"""Wire-protocol server throughput over loopback:
N concurrent clients send the reference recovery request (corrupted plane +
all k references, recovery.py:219-227) for 720p RGB and depth; frames/s with
max_connections=1 (the reference's serial server) vs concurrent pinned
connections.  Prints one JSON line per setting."""
import json
import os
import socket
import struct
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_2604_27441_b200 import Checkpoint, ModelConfig  # noqa: E402
from paper_2604_27441_b200.server import MSG_REQUEST, RecoveryServer  # noqa: E402

H, W, K = 720, 1280, 5


def make_request(mod, rng):
    c = 3 if mod == 0 else 1
    planes = rng.integers(0, 256, (K + 1, H, W, c), dtype=np.uint8)
    grid = rng.random((H // 16, W // 16)) < 0.01
    body = struct.pack("<BBIHHB", MSG_REQUEST, mod, 1, W, H, K)
    body += np.packbits(grid.reshape(-1)).tobytes() + planes.tobytes()
    return struct.pack("<I", len(body)) + body, H * W * c


def recv_exact(sock, n, buf):
    view = memoryview(buf)[:n]
    got = 0
    while got < n:
        k = sock.recv_into(view[got:])
        if not k:
            raise ConnectionError("closed")
        got += k


def run(max_conn, clients, seconds):
    ck = {c: Checkpoint.random_init(ModelConfig(), c, seed=0) for c in (3, 1)}
    srv = RecoveryServer(("127.0.0.1", 0), checkpoint_rgb=ck[3], checkpoint_depth=ck[1],
                         max_connections=max_conn)
    srv.start()
    rng = np.random.default_rng(0)
    reqs = [make_request(m, rng) for m in (0, 1)]
    done = [0] * clients
    stop = time.perf_counter() + seconds

    def client(i):
        s = socket.create_connection(srv.addr)
        s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
        head = bytearray(8)
        recv_exact(s, 4, head)
        (n,) = struct.unpack("<I", head[:4])
        recv_exact(s, n, bytearray(n))
        out = bytearray(H * W * 3 + 16)
        while time.perf_counter() < stop:
            for payload, nplane in reqs:
                s.sendall(payload)
                recv_exact(s, 4, head)
                (n,) = struct.unpack("<I", head[:4])
                recv_exact(s, n, out)
            done[i] += 1
        s.close()

    t0 = time.perf_counter()
    th = [threading.Thread(target=client, args=(i,)) for i in range(clients)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    el = time.perf_counter() - t0
    srv.close()
    return sum(done) / el


if __name__ == "__main__":
    for mc, cl in ((1, 4), (8, 4)):
        fps = run(mc, cl, 6.0)
        print(json.dumps({"metric": "RGB-D frames/s through the TCP recovery protocol (720p, k=5 "
                                    "refs per request, loopback)", "max_connections": mc,
                          "clients": cl, "value": fps}), flush=True)
