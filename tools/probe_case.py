import os, sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from golden_cases import recover_case
from helpers import GOLDEN_DIR
import torch
import paper_2604_27441_b200 as p
from paper_2604_27441_b200.recovery import RecoveryEngine
RECOV = np.load(os.path.join(GOLDEN_DIR, "recover_golden.npz"))
for name in sorted(n for n in RECOV.files if "__" not in n):
    arch, c, state, plane, grid, refs = recover_case(name)
    for prec in ("fast", "precise"):
        cfg = p.ModelConfig(k=arch.k, tubelet_t=arch.tubelet_t, patch=arch.patch, dim=arch.dim, layers=arch.layers, heads=arch.heads)
        m = p.MaskedVideoModel(cfg, c, precision=prec)
        m.load_state_dict({k: torch.from_numpy(v) for k, v in state.items()})
        got = RecoveryEngine(m, prec).recover(plane, grid, refs)
        d = np.abs(got.astype(int) - RECOV[name].astype(int))
        print(name, prec, "masked", int(grid.sum()), "maxdiff", d.max(), "n>2", int((d > 2).sum()))
