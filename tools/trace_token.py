"""Phase timeline of CTA 0 / slot 0 of the three precise block-tail phase
kernels (token_x3_kernel<0,1,2>), first two tiles, from the NVREC_TRACE build:

    make -C paper_2604_27441_b200/csrc TRACE=1
    NVREC_LIB=paper_2604_27441_b200/lib/libnvrec_b200_trace.so python tools/trace_token.py
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

NAMES = {0: ["start", "ao loaded", "proj_s mma", "LN_t", "qkv_t mma", "attn_t", "proj_t mma"],
         1: ["start", "x loaded", "LN_m", "fc1 h0 mma", "GELU0", "fc2/fc1 h1 mma", "GELU1", "fc2 mma"],
         2: ["start", "x loaded", "LN_s", "qkv_s mma"]}
prec = sys.argv[1] if len(sys.argv) > 1 else "precise"
dev = torch.device("cuda", 0)
wl = bench.Workload("trace", 720, 1280, range(8), ("ge",))
wk = bench.ModalityWork(wl, "rgb", 3, 1024, dev, prec)
st = torch.cuda.current_stream(dev)
for _ in range(3):
    wk.device_step(st)
torch.cuda.synchronize()
lib = _native.load_library()
if prec == "fast":
    # fused fast tail (token_tc_kernel), CTA 0 / slot 0, first two tiles
    fb = (ctypes.c_ulonglong * 32)()
    lib.nvrec_debug_token_tc_trace(fb, 32)
    ft = np.frombuffer(fb, dtype=np.uint64).astype(np.int64).reshape(2, 16)
    names = ["start", "ao/x loaded", "proj_s mma", "LN_t", "qkv_t mma", "attn_t", "proj_t mma",
             "LN_m", "fc1 mma", "GELU stored", "fc2 mma", "x stored + LN_s", "qkv_s mma"]
    for t in range(2):
        e = ft[t]
        row = ["%s +%d" % (names[i], e[i] - e[i - 1]) for i in range(1, len(names))]
        print("token_tc tile %d: total %d | %s | end +%d" % (t, e[15] - e[0], ", ".join(row),
                                                          e[15] - e[12]))
    sys.exit(0)
buf = (ctypes.c_ulonglong * 96)()
lib.nvrec_debug_token_x3_trace(buf, 96)
tr = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(3, 2, 16)
for ph in range(3):
    for t in range(2):
        e = tr[ph, t]
        names = NAMES[ph]
        row = ["%s +%d" % (names[i], e[i] - e[i - 1]) for i in range(1, len(names)) if e[i] and e[i - 1]]
        print("phase %d tile %d: total %d | %s | end +%d" % (ph, t, e[15] - e[0], ", ".join(row),
                                                           e[15] - e[len(names) - 1]))
