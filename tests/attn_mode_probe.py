"""Helper for test_gpu_parity.test_speculative_max_*: one recovery (and one
forward with sharply scaled attention scores) at precision argv[2] under the
NVREC_ATTN_MODE chosen by the parent; writes the outputs to argv[1]."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_27441_b200 import Checkpoint, ModelConfig  # noqa: E402
from paper_2604_27441_b200.recovery import RecoveryEngine  # noqa: E402

prec = sys.argv[2] if len(sys.argv) > 2 else "fast"
ck = Checkpoint.random_init(ModelConfig(), 3, seed=7)
rng = np.random.default_rng(7)
frames = rng.integers(0, 256, (6, 240, 320, 3), dtype=np.uint8)
grid = rng.random((15, 20)) < 0.3
out = RecoveryEngine(ck.build_model(precision=prec), prec).recover(frames[-1], grid,
                                                                 list(frames[:-1]))
# sharp scores: scale the spatial q/k projections so the running max jumps by
# hundreds (log2 units) between key tiles and the speculative exponent overflows
state = {k: v.clone() for k, v in ck.state.items()}
for i in range(2):
    w = state["blocks.%d.attn_s.qkv.weight" % i]
    w[:128] *= 60.0
ck2 = Checkpoint(ck.config, ck.channels, state)
model = ck2.build_model(precision=prec)
stack = torch.rand(1, 6, 3, 240, 320, generator=torch.Generator().manual_seed(3)).cuda()
mask = torch.from_numpy(rng.random((1, 240, 320)) < 0.3).cuda()
from paper_2604_27441_b200 import _native  # noqa: E402
before = _native.attn_fixup_items()
sharp = model(stack, mask).cpu().numpy()
redone = _native.attn_fixup_items() - before
# moderately sharp scores: later key tiles exceed the speculative max by a few
# log2 units, so the in-kernel rescale of P (and of the accumulated O) runs
# without overflowing into the fix-up
moderate = []
for f in (2.0, 3.0, 4.0):
    st2 = {k: v.clone() for k, v in ck.state.items()}
    for i in range(2):
        st2["blocks.%d.attn_s.qkv.weight" % i][:128] *= f
    m2 = Checkpoint(ck.config, ck.channels, st2).build_model(precision=prec)
    moderate.append(m2(stack, mask).cpu().numpy())
np.savez(sys.argv[1], out=out, sharp=sharp, redone=redone, moderate=np.stack(moderate))
