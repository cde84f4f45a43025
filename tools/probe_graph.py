"""Device step with and without a CUDA graph around both modalities (diagnostic)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench

dev = torch.device("cuda", 0)
works = [bench.ModalityWork(n, c, L, list(range(8)), device=dev, precision="fast")
         for n, c, L in bench.MODS]
streams = [torch.cuda.Stream(dev) for _ in works]
bench.run_steps(works, streams, "device_step", 5)
torch.cuda.synchronize()
ms = bench.timed(works, streams, "device_step", 100, False)
print("eager   %.3f ms/step  %.0f frames/s" % (ms / 100, 8 * 100 / (ms / 1000)))
g = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream(dev)
cap.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=cap):
    ev = cap.record_event()
    for wk, st in zip(works, streams):
        st.wait_event(ev)
        with torch.cuda.stream(st):
            wk.device_step(st)
    for st in streams:
        cap.wait_stream(st)
torch.cuda.synchronize()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(100):
    g.replay()
t1.record()
torch.cuda.synchronize()
ms = t0.elapsed_time(t1)
print("graph   %.3f ms/step  %.0f frames/s" % (ms / 100, 8 * 100 / (ms / 1000)))
