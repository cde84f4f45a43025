"""H2D bandwidth: one cudaMemcpyAsync vs chunks over several streams, and a
kernel reading mapped pinned memory (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch

dev = torch.device("cuda", 0)
N = int(29.5e6)
x = torch.empty(N, dtype=torch.uint8).pin_memory()
y = torch.empty(N, dtype=torch.uint8, device=dev)
streams = [torch.cuda.Stream(dev) for _ in range(8)]


def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


for ns in (1, 2, 4, 8):
    def f(ns=ns):
        ch = (N + ns - 1) // ns
        for k in range(ns):
            with torch.cuda.stream(streams[k]):
                y[k * ch:(k + 1) * ch].copy_(x[k * ch:(k + 1) * ch], non_blocking=True)
        for k in range(ns):
            torch.cuda.current_stream().wait_stream(streams[k])
    ms = t(f)
    print("H2D %d streams: %.3f ms  %.1f GB/s" % (ns, ms, N / ms / 1e6), flush=True)
for ns in (1, 2, 4):
    def g(ns=ns):
        ch = (N + ns - 1) // ns
        for k in range(ns):
            with torch.cuda.stream(streams[k]):
                x[k * ch:(k + 1) * ch].copy_(y[k * ch:(k + 1) * ch], non_blocking=True)
        for k in range(ns):
            torch.cuda.current_stream().wait_stream(streams[k])
    ms = t(g)
    print("D2H %d streams: %.3f ms  %.1f GB/s" % (ns, ms, N / ms / 1e6), flush=True)
# both directions at once
def both():
    with torch.cuda.stream(streams[0]):
        y.copy_(x, non_blocking=True)
    z = torch.empty_like(x)
    with torch.cuda.stream(streams[1]):
        pass
ms = t(lambda: [y.copy_(x, non_blocking=True)])
import subprocess
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:1500])
print(subprocess.run(["nvidia-smi", "-q", "-d", "PCIE"], capture_output=True, text=True).stdout[:2500])
