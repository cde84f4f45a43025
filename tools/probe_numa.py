"""Host placement probe: the GPU's local CPUs (NVML), the NUMA nodes, and
H2D/D2H bandwidth of pinned buffers allocated with and without pinning the
process to those CPUs first (diagnostic for the e2e spread across boxes)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.getcwd())


def local_cpus():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    n = os.cpu_count()
    words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
    cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
    return [c for c in cpus if c < n]


def bw(tag):
    dev = torch.device("cuda", 0)
    N = int(29.5e6)
    x = torch.empty(N, dtype=torch.uint8).pin_memory()
    x.fill_(1)
    y = torch.empty(N, dtype=torch.uint8, device=dev)
    st = [torch.cuda.Stream(dev) for _ in range(4)]

    def run(h2d):
        ch = N // 4
        for k in range(4):
            with torch.cuda.stream(st[k]):
                if h2d:
                    y[k * ch:(k + 1) * ch].copy_(x[k * ch:(k + 1) * ch], non_blocking=True)
                else:
                    x[k * ch:(k + 1) * ch].copy_(y[k * ch:(k + 1) * ch], non_blocking=True)
        torch.cuda.synchronize()

    for h2d in (True, False):
        run(h2d)
        t0 = time.perf_counter()
        for _ in range(20):
            run(h2d)
        ms = (time.perf_counter() - t0) / 20 * 1e3
        print("%s %s %.1f GB/s" % (tag, "H2D" if h2d else "D2H", N / ms / 1e6), flush=True)


print("cpus", os.cpu_count(), "affinity now", len(os.sched_getaffinity(0)))
try:
    print("numa nodes", sorted(os.listdir("/sys/devices/system/node")))
except OSError:
    pass
cpus = local_cpus()
print("gpu-local cpus", len(cpus), cpus[:8], "...")
bw("default")
os.sched_setaffinity(0, cpus)
bw("gpu-local")
