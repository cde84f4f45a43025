"""Phase timeline of one CTA of the dense precise attention kernel
(attn_x3w_kernel), from the NVREC_TRACE build:

    make -C paper_2604_27441_b200/csrc TRACE=1
    NVREC_LIB=paper_2604_27441_b200/lib/libnvrec_b200_trace.so python tools/trace_attn.py

Softmax events per key tile j: 0 wait S / 1 S ready / 2 chunk 0 stored /
3 O' folded / 4 chunk 1 stored / 5 P arrived.  MMA issuer per S tile n:
0 start / 1 S issued / 2 P(n-2) ready / 3 PV issued."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2604_27441_b200 import _native  # noqa: E402

dev = torch.device("cuda", 0)
wl = bench.Workload("trace", 720, 1280, range(8), ("ge",))
wk = bench.ModalityWork(wl, "rgb", 3, 1024, dev, "precise")
st = torch.cuda.current_stream(dev)
for _ in range(3):
    wk.device_step(st)
torch.cuda.synchronize()
lib = _native.load_library()
buf = (ctypes.c_ulonglong * (3 * 128 * 8))()
n = lib.nvrec_debug_attn_trace(buf, 3 * 128 * 8)
tr = np.frombuffer(buf, dtype=np.uint64).reshape(3, 128, 8).astype(np.int64)
t0 = tr[tr > 0].min()
rel = np.where(tr > 0, tr - t0, -1)
for role, name in ((0, "tile0"), (1, "tile1")):
    print("== softmax", name, "  (cycles: wait_S, chunk0, fold, chunk1, tail; start)")
    for j in range(30):
        e = rel[role, j]
        if e[0] < 0:
            break
        print("j=%2d start %7d  waitS %5d  c0 %5d  fold %5d  c1 %5d  tail %5d" %
              (j, e[0], e[1] - e[0], e[2] - e[1], e[3] - e[2], e[4] - e[3], e[5] - e[4]))
print("== MMA issuer  (S issue, wait P, PV issue; start)")
for i in range(62):
    e = rel[2, i]
    if e[0] < 0:
        break
    print("n=%2d start %7d  S %5d  waitP %5d  PV %5d" %
          (i, e[0], e[1] - e[0], (e[2] - e[1]) if e[2] >= 0 else -1,
           (e[3] - e[2]) if e[2] >= 0 else e[3] - e[1]))
