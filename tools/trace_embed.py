"""Stage timeline of CTA (0,0,0) of the u8 tensor-core embedding (RGB, the
bench's precision) from the NVREC_TRACE build: per K stage the MMA thread's
waits for the converted A operand and the weight block, the converters' wait
for the raw pixels; then the epilogue phases.

    make -C paper_2604_27441_b200/csrc TRACE=1
    NVREC_LIB=paper_2604_27441_b200/lib/libnvrec_b200_trace.so python tools/trace_embed.py [fast]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2604_27441_b200 import _native  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "precise"
dev = torch.device("cuda", 0)
wl = bench.Workload("trace", 720, 1280, range(8), ("ge",))
wk = bench.ModalityWork(wl, "rgb", 3, 1024, dev, prec)
st = torch.cuda.current_stream(dev)
for _ in range(3):
    wk.device_step(st)
torch.cuda.synchronize()
lib = _native.load_library()
buf = (ctypes.c_ulonglong * 264)()
lib.nvrec_debug_embed_trace(buf, 264)
tr = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
stg, end = tr[:256].reshape(64, 4), tr[256:264]
t0 = stg[0, 0]
prev = t0
for i in range(64):
    if stg[i, 0] == 0:
        break
    print("stage %2d start %6d  waitA %5d  waitW %5d  pixels@ %6d  (+%d since prev)" % (
        i, stg[i, 0] - t0, stg[i, 1] - stg[i, 0], stg[i, 2] - stg[i, 1], stg[i, 3] - t0,
        stg[i, 0] - prev))
    prev = stg[i, 0]
names = ["epi wait acc", "acc ready", "A2 stored", "qkv ready", "stores done", "all done"]
for i, n in enumerate(names):
    print("%-14s %7d" % (n, end[i] - t0))
