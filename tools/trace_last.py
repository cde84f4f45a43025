"""Phase timeline of CTA 0 of the tensor-core last block (last_tc_kernel) from
the NVREC_TRACE build, headline workload (8 x 720p RGB, GE loss or --loss):

    make -C paper_2604_27441_b200/csrc TRACE=1
    NVREC_LIB=paper_2604_27441_b200/lib/libnvrec_b200_trace.so python tools/trace_last.py [block:0.2]
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

NAMES = ["start", "setup", "ao loaded", "proj_s done", "LN_t done", "qkv_t done", "attn_t done",
         "proj_t done", "LN_m done", "fc1 h0 done", "GELU0 stored", "fc2/fc1 h1 done",
         "GELU1 stored", "fc2 done", "final LN", "head0 mma", "head0 epi", "head1 mma",
         "head1 epi", "head2 mma", "head2 epi", "head3 mma", "head3 epi", "tile end"]
loss = ("ge",) if len(sys.argv) < 2 else (sys.argv[1].split(":")[0], float(sys.argv[1].split(":")[1]))
dev = torch.device("cuda", 0)
wl = bench.Workload("trace", 720, 1280, range(8), loss)
wk = bench.ModalityWork(wl, "rgb", 3, 1024, dev, "precise")
st = torch.cuda.current_stream(dev)
for _ in range(3):
    wk.device_step(st)
torch.cuda.synchronize()
lib = _native.load_library()
buf = (ctypes.c_ulonglong * 64)()
lib.nvrec_debug_last_trace(buf, 64)
tr = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)[:len(NAMES)]
prev = tr[0]
for i, nm in enumerate(NAMES):
    print("%2d %-18s %8d  +%6d" % (i, nm, tr[i] - tr[0], tr[i] - prev))
    prev = tr[i]
