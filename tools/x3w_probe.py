"""Dense precise attention A/B: 64-key kernel (NVREC_ATTN_X3W=0 in a child) vs
attn_x3w_kernel against the oracle on one RGB frame of size argv[1] x argv[2]."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

h, w = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3:
    import torch
    from helpers import block_grid, make_state, textured_u8
    from oracle import nvrec_forward
    from paper_2604_27441_b200 import MaskedVideoModel, ModelConfig, _native
    from paper_2604_27441_b200.recovery import RecoveryEngine
    arch = nvrec_forward.Arch()
    rng = np.random.default_rng(720 + 3)
    state = make_state(arch, 3, 7200 + 3)
    frames = textured_u8(rng, 6, h, w, 3)
    grid = block_grid(rng, h // 16, w // 16, 0.1)
    m = MaskedVideoModel(ModelConfig(), 3, precision="precise")
    m.load_state_dict({k: torch.from_numpy(v) for k, v in state.items()})
    before = _native.attn_fixup_items()
    got = RecoveryEngine(m, "precise").recover(frames[-1], grid, list(frames[:-1]))
    np.savez(sys.argv[3], got=got, redone=_native.attn_fixup_items() - before)
    sys.exit(0)
from helpers import block_grid, make_state, textured_u8  # noqa: E402
from oracle import nvrec_forward, recover as oracle_recover  # noqa: E402
arch = nvrec_forward.Arch()
rng = np.random.default_rng(720 + 3)
state = make_state(arch, 3, 7200 + 3)
frames = textured_u8(rng, 6, h, w, 3)
grid = block_grid(rng, h // 16, w // 16, 0.1)
want = oracle_recover.recover(state, arch, 3, frames[-1], grid, list(frames[:-1]))
for flag in ("0", "1"):
    subprocess.run([sys.executable, __file__, str(h), str(w), "/tmp/x3w.npz"], check=True,
                   env=dict(os.environ, NVREC_ATTN_X3W=flag), timeout=120)
    r = np.load("/tmp/x3w.npz")
    d = np.abs(r["got"].astype(int) - want.astype(int))
    print("x3w=%s %dx%d maxdiff %d n>1 %d redone %d" % (flag, h, w, d.max(), int((d > 1).sum()),
                                                       int(r["redone"])), flush=True)
