"""Module API (float stacks) forward of 8 x 720p RGB and depth, for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_27441_b200 import Checkpoint, ModelConfig  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "precise"
for c in (3, 1):
    m = Checkpoint.random_init(ModelConfig(), c, seed=0).build_model(precision=prec)
    g = torch.Generator(device="cpu").manual_seed(5)
    stack = torch.rand(8, 6, c, 720, 1280, generator=g).cuda()
    mask = (torch.rand(8, 720, 1280, generator=g) < 0.1).cuda()
    for _ in range(2):
        m(stack, mask)
torch.cuda.synchronize()
print("ok")
