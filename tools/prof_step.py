"""Profiling driver: the headline bench step (8 x 720p RGB-D streams, GE
loss) run N times with inputs resident, for ncu / compute-sanitizer.

    python tools/prof_step.py [--precision precise|fast] [--steps 3] [--streams 8]
                              [--loss ge|block:0.2] [--h 720 --w 1280]
"""
from __future__ import annotations

import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="precise")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--streams", type=int, default=8)
    ap.add_argument("--loss", default="ge")
    ap.add_argument("--h", type=int, default=720)
    ap.add_argument("--w", type=int, default=1280)
    ap.add_argument("--serial", action="store_true", help="both modalities on one stream")
    a = ap.parse_args()
    loss = ("ge",) if a.loss == "ge" else (a.loss.split(":")[0], float(a.loss.split(":")[1]))
    dev = torch.device("cuda", 0)
    wl = bench.Workload("prof", a.h, a.w, range(a.streams), loss)
    works = [bench.ModalityWork(wl, n, c, L, dev, a.precision) for n, c, L in bench.MODS]
    streams = [torch.cuda.current_stream(dev)] * 2 if a.serial else \
        [torch.cuda.Stream(dev) for _ in works]
    bench.run_steps(works, streams, "device_step", a.steps)
    torch.cuda.synchronize()
    print("ok", [w.masked_patches[:4] for w in works])


if __name__ == "__main__":
    main()
