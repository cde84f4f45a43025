"""One u8 recovery per (modality, precision) named on the command line, for
compute-sanitizer runs: python tools/sync_probe.py 1:fast 3:precise ..."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_27441_b200 import Checkpoint, ModelConfig  # noqa: E402
from paper_2604_27441_b200.recovery import RecoveryEngine  # noqa: E402

rng = np.random.default_rng(0)
for arg in sys.argv[1:]:
    c, prec = arg.split(":")
    c = int(c)
    ck = Checkpoint.random_init(ModelConfig(), c, seed=c)
    frames = rng.integers(0, 256, (6, 64, 96, c), dtype=np.uint8)
    grid = rng.random((4, 6)) < 0.3
    grid[0, 0] = True
    RecoveryEngine(ck.build_model(precision=prec), prec).recover(frames[-1], grid, list(frames[:-1]))
    print(arg, "ok", flush=True)
