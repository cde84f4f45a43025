"""Helper for test_gpu_parity.test_last_block_tc_equals_simt: a batched u8
recovery (streams with 0 %, 5 %, 20 %, 60 % and 100 % masked patches, so the
gathered last-block tiles straddle streams and skip empty ones) and a dense
float forward, per precision and modality, under the NVREC_LAST_SIMT chosen by
the parent; writes the outputs to argv[1]."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_27441_b200 import Checkpoint, ModelConfig, _native  # noqa: E402
from paper_2604_27441_b200.recovery import RecoveryEngine, pack_grid, stack_slots  # noqa: E402

out = {}
h, w = 240, 320
for c in (3, 1):
    ck = Checkpoint.random_init(ModelConfig(), c, seed=40 + c)
    rng = np.random.default_rng(40 + c)
    dens = (0.0, 0.05, 0.2, 0.6, 1.0)
    B = len(dens)
    frames = torch.from_numpy(rng.integers(0, 256, (6 * B, h, w, c), dtype=np.uint8)).cuda()
    idx = torch.tensor([[6 * s + i for i in stack_slots(5, 5, 6)] for s in range(B)],
                       dtype=torch.int32).cuda()
    bits = torch.from_numpy(np.stack([pack_grid(rng.random((h // 16, w // 16)) < p)
                                      for p in dens])).cuda()
    stack = torch.rand(2, 6, c, h, w, generator=torch.Generator().manual_seed(c)).cuda()
    mask = torch.from_numpy(rng.random((2, h, w)) < 0.3).cuda()
    for prec in ("fast", "precise"):
        model = ck.build_model(precision=prec)
        eng = RecoveryEngine(model, prec)
        with _native.StageProfile() as prof:
            out["u8_%d_%s" % (c, prec)] = eng.recover_device(frames, idx, bits).cpu().numpy()
            torch.cuda.synchronize()
        out["last_tc_%d_%s" % (c, prec)] = prof.launches["last_tc"]
        out["f32_%d_%s" % (c, prec)] = model(stack, mask).cpu().numpy()
np.savez(sys.argv[1], **out)
