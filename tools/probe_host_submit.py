"""Host-side cost of one pipeline submit (Python staging + launches), per
modality, for the receiver and the plane-in pipelines (diagnostic)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402

dev = torch.device("cuda", 0)
works = [bench.ModalityWork(n, c, L, list(range(8)), device=dev, precision="fast") for n, c, L in bench.MODS]
rworks = [bench.ReceiverWork(n, c, L, list(range(8)), dev, wk.engine)
          for (n, c, L), wk in zip(bench.MODS, works)]
for _ in range(6):
    for rw in rworks:
        rw.submit()
    for wk in works:
        wk.pipe.submit(None, wk.jobs)
torch.cuda.synchronize()
for name, fn in (("receiver", lambda: [rw.submit() for rw in rworks]),
                 ("planes", lambda: [wk.pipe.submit(None, wk.jobs) for wk in works])):
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    ts.sort()
    print("%s submit (both modalities): median %.3f ms, min %.3f ms" % (name, ts[15] * 1e3, ts[0] * 1e3))
from paper_2604_27441_b200.codec import DecodeBatch  # noqa: E402
rw = rworks[0]
items = None
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    rw.submit()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
