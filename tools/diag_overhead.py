"""Host-overhead diagnostic: wall time per recover_device call vs device time."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_27441_b200 import Checkpoint, ModelConfig, _native
from paper_2604_27441_b200.recovery import RecoveryEngine, pack_grid, stack_slots

dev = torch.device("cuda", 0)
for c in (3, 1):
    ck = Checkpoint.random_init(ModelConfig(), c, seed=0)
    eng = RecoveryEngine(ck.build_model(), "fast")
    H, W, B = 720, 1280, int(sys.argv[1]) if len(sys.argv) > 1 else 1
    frames = torch.randint(0, 256, (6 * B, H, W, c), dtype=torch.uint8, device=dev)
    idx = torch.tensor([[6 * s + i for i in stack_slots(5, 5, 6)] for s in range(B)],
                       dtype=torch.int32, device=dev)
    rng = np.random.default_rng(0)
    bits = torch.from_numpy(np.stack([pack_grid(rng.random((45, 80)) < 0.1) for _ in range(B)])).to(dev)
    out = torch.empty((B, H, W, c), dtype=torch.uint8, device=dev)
    for _ in range(3):
        eng.recover_device(frames, idx, bits, out)
    torch.cuda.synchronize()
    for trial in range(3):
        t0 = time.perf_counter()
        eng.recover_device(frames, idx, bits, out)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print("c=%d B=%d host call %.3f ms, call+sync %.3f ms" % (c, B, 1e3 * (t1 - t0), 1e3 * (t2 - t0)))
    with _native.StageProfile() as prof:
        eng.recover_device(frames, idx, bits, out)
        torch.cuda.synchronize()
    print({k: round(v, 3) for k, v in prof.ms.items() if v})
