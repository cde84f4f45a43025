"""Pipeline diagnostics: wall time per step of RecoveryPipeline.submit with
copies / graphs toggled (not a bench number)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench

dev = torch.device("cuda", 0)
works = [bench.ModalityWork(n, c, L, list(range(8)), device=dev, precision="fast")
         for n, c, L in bench.MODS]


def run(label, n=60):
    for wk in works:
        for _ in range(6):
            wk.pipe.submit(None, wk.jobs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        for wk in works:
            wk.pipe.submit(None, wk.jobs)
    torch.cuda.synchronize()
    print("%-28s %.3f ms/step" % (label, (time.perf_counter() - t0) / n * 1e3), flush=True)


run("default (graphs, copies)")
for wk in works:
    wk.pipe.use_graphs = False
run("no graphs")
for wk in works:
    wk.pipe.use_graphs = True
# drop the plane H2D / D2H by shrinking them to one row
orig = []
for wk in works:
    p = wk.pipe
    orig.append((p.host_in, p.host_out, p.frames))
import types
def submit_nocopy(self, planes, frames, h2d=True, d2h=True):
    i = self.step % self.nbuf
    if self.step >= self.nbuf:
        self.ev_h2d[i].synchronize(); self.ev_d2h[i].synchronize()
    self.lm[i].stage(frames)
    hd = self.head
    if self.step >= self.nbuf:
        self.s_h2d.wait_event(self.ev_cmp[i])
    with torch.cuda.stream(self.s_h2d):
        if h2d:
            self.frames[self.k + i].copy_(self.host_in[i], non_blocking=True)
        self.lm[i].dev_in.copy_(self.lm[i].host, non_blocking=True)
        self.ev_h2d[i].record(self.s_h2d)
    self.s_cmp.wait_event(self.ev_h2d[i])
    if self.ev_slot[hd] is not None:
        self.s_cmp.wait_event(self.ev_slot[hd])
    self._run(hd, i)
    self.ev_cmp[i].record(self.s_cmp)
    self.s_d2h.wait_event(self.ev_cmp[i])
    with torch.cuda.stream(self.s_d2h):
        if d2h:
            self.host_out[i].copy_(self.frames[hd], non_blocking=True)
        self.ev_d2h[i].record(self.s_d2h)
    self.ev_slot[hd] = self.ev_d2h[i]
    self.head = (hd + 1) % self.k
    self.step += 1
    return i
for flags, label in (((False, True), "no plane H2D"), ((True, False), "no D2H"),
                     ((False, False), "no plane copies")):
    for wk in works:
        wk.pipe.submit = types.MethodType(lambda self, pl, fr, f=flags: submit_nocopy(self, pl, fr, *f), wk.pipe)
    run(label)
# raw copy bandwidth
x = torch.empty(int(29.5e6), dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device=dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
print("H2D 29.5 MB: %.3f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
t0 = time.perf_counter()
for _ in range(20):
    x.copy_(y, non_blocking=True)
torch.cuda.synchronize()
print("D2H 29.5 MB: %.3f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
