"""Benchmark: recovered 1280x720 RGB-D frames/s per GPU (+ p50 latency).

Headline workload (BASELINE.json configs[2] x configs[4]): each GPU serves S
independent 720p RGB-D conference streams (default 8, so 8 GPUs = the
64-stream multi-party config; weak scaling, no collective on the data
path).  One step = one frame of every stream, both modalities:

  loss mask   synthetic codec P-frame headers (~10% changed blocks) whose
              body shards are dropped by a Gilbert-Elliott channel
              (p_gb=0.0155, p_bg=0.5, tests/test_acceptance.py:263-264)
              -> nvrec_loss_mask (bit-exact receiver+codec mask)
  recovery    nvrec_recover_u8 over the S streams of each modality (RGB and
              depth on two CUDA streams): u8 stack of 5 references + the
              corrupted plane, model forward, quantise, masked merge.

Arithmetic: ``--precision precise`` (the default and the headline) is
fp32-class -- every tensor-core product from split operands (a = hi + lo,
hi*hi + hi*lo + lo*hi, fp32 accumulation; 720p max-abs ~5e-7 against the
reference's fp32 forward); the ``fast`` path (bf16/fp16 operands) is
measured beside it.

``value`` = frames/s with inputs resident in HBM (device-timed, CUDA
events, max over ranks).  ``e2e`` = the same step through host buffers
(RecoveryPipeline): pinned H2D of every stream's new corrupted plane and
loss-mask job, recovery on the device-resident reference rings, D2H of the
recovered planes, inside the timed region.  ``configs`` holds the other
BASELINE.json shapes and mask densities (320x240, 640x480, 720p at 10% and
20% block loss, 1920x1088 at 20%, 64 streams on one GPU).

``--impl reference`` times the reference CPU path (the oracle restatement
of the receiver's loss mask and RecoveryServer._recover in fp32 torch-CPU
ops -- the same ATen kernels the reference module calls) on the host cores,
rank 0 only, on the SAME synthetic inputs as the GPU arm: the same streams'
planes, the same GE-dropped shards, the same random-init weights; each step
is one stream's RGB-D frame (a bounded sample of the 8-stream step).

``--gpus N`` without torchrun re-launches itself under torch.distributed.run
with N ranks (127.0.0.1).  ``--dry-run`` exercises only the launch / timing
/ reporting logic (gloo, no GPU work; used by the CPU tests).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, W = 720, 1280
METRIC = "recovered RGB-D frames/sec/GPU and p50 per-frame latency at 720p"
MODS = (("rgb", 3, 1024), ("depth", 1, 512))      # name, channels, shard L
MUFU_PEAK = 148 * 16 * 1.965e9                      # ex2/s, derived
PRECISE_DTYPE = "f32"
PRECISE_NOTE = ("fp32-class: every tensor-core product from split operands (bf16 hi/lo for "
                "attention Q/K/V/P, fp16 hi/lo with per-matrix 2^s pre-scale for the weights "
                "and activations of the embed/linear GEMMs), hi*hi + hi*lo + lo*hi with fp32 "
                "accumulation; softmax, LayerNorm, GELU, residual, head fp32; measured 720p "
                "max-abs 4.8e-7 (RGB) / 5.7e-7 (depth) vs the reference's fp32 forward")
WORKLOAD_720P = ("1280x720 RGB-D streams (configs[2] x configs[4]): %d streams/GPU, GE loss "
                 "(p_gb=0.0155,p_bg=0.5) on body shards of synthetic P-frame headers (~10%% "
                 "changed blocks), k=5 refs, random-init weights (seed 0)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--streams-per-gpu", type=int, default=8)
    ap.add_argument("--precision", default="precise", choices=["fast", "precise"])
    ap.add_argument("--latency-iters", type=int, default=50)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the fast-path, other-config and density lines")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch/timing/report logic only (gloo, no GPU work)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


def spawn_ranks(args) -> None:
    """``--gpus N`` outside torchrun: re-run this script with N ranks."""
    if args.gpus <= 1 or "RANK" in os.environ:
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def max_over_ranks(ms: float, dist_on: bool, device=None) -> float:
    if not dist_on:
        return ms
    t = torch.tensor([ms], device=device) if device is not None else torch.tensor([ms])
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------
# clocks sampled DURING the timed region (NVML thread, 2 ms period)

class ClockSampler:
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
               "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int, period_s: float = 0.002):
        self.sm, self.reasons, self.mx = [], set(), None
        self.stop_ev = threading.Event()
        self.err = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001 -- report, do not fail the bench
            self.nv, self.err = None, repr(e)
        self.period = period_s
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception as e:  # noqa: BLE001
                self.err = repr(e)
                return
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self.th.start()
        return self

    def __exit__(self, *exc):
        self.stop_ev.set()
        if self.nv is not None:
            self.th.join()
        return False

    def result(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable: %s" % self.err]}
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "NVML every 2 ms during the timed device region"}


# ----------------------------------------------------------------------------
# synthetic inputs, shared by the GPU arm and the reference (CPU) arm

def stream_planes(c: int, h: int, w: int, sid: int, F: int = 6) -> np.ndarray:
    """(F, h, w, c) u8: a random 8x8-block texture drifting one pixel per
    frame (5 references + the corrupted plane of stream ``sid``)."""
    rng = np.random.default_rng(1000 * c + 7919 * sid)
    base = rng.integers(0, 256, (h // 8 + 2, w // 8 + 2, c), dtype=np.uint8)
    tex = np.kron(base, np.ones((8, 8, 1), np.uint8))
    return np.stack([tex[i % 8: i % 8 + h, 0:w] for i in range(F)])


def stream_planes16(h: int, w: int, sid: int, F: int = 6) -> np.ndarray:
    """(F, h, w) u16 depth: 8x8-block depth steps (300..9000 units) drifting
    one pixel per frame, slowly receding."""
    rng = np.random.default_rng(16000 + 7919 * sid)
    base = rng.integers(300, 9000, (h // 8 + 2, w // 8 + 2)).astype(np.uint16)
    tex = np.kron(base, np.ones((8, 8), np.uint16))
    return np.stack([tex[i % 8: i % 8 + h, 0:w] + np.uint16(3 * i) for i in range(F)])


class Workload:
    """One BASELINE config: resolution, streams, and how a stream's loss mask
    arises -- ``("ge",)`` Gilbert-Elliott body-shard loss, ``("bern", p)``
    Bernoulli shard loss (both through the receiver/codec mask), or
    ``("block", r)`` a synthetic block mask (nvrec data.synthetic_mask)."""

    def __init__(self, name, h, w, stream_ids, loss=("ge",), depth16=False):
        self.name, self.h, self.w, self.loss = name, h, w, loss
        self.ids = list(stream_ids)
        self.depth16 = depth16          # depth as u16 planes (nvrec_recover_u16)

    def planes(self, c, sid):
        return stream_planes(c, self.h, self.w, sid)

    def job(self, c, L, s, sid):
        """(header, n_data, received, encoded_len) for mask kinds ge/bern."""
        from tools.synth import GilbertElliott, p_frame_shards
        rng = np.random.default_rng(sid + c)
        if self.loss[0] == "ge":
            drop = GilbertElliott(seed=sid + 17 * c).drop
        else:
            lrng = np.random.default_rng(50000 + sid + 17 * c)
            drop = (lambda: bool(lrng.random() < self.loss[1]))
        hdr, nd, recv, enc = p_frame_shards(rng, self.w, self.h, c, L, drop, present_ratio=0.1)
        if recv.all():                     # every stream needs recovery
            recv[1 + (s % max(1, nd - 1))] = False
        return hdr, nd, recv, enc

    def grid(self, c, sid):
        """Block grid for mask kind ``block``."""
        from paper_2604_27441_b200.data import synthetic_mask
        rng = np.random.default_rng(90000 + sid + 17 * c)
        m = synthetic_mask(self.h, self.w, self.loss[1], rng)
        g = m[::16, ::16].copy()
        if not g.any():
            g[0, 0] = True
        return g

    def describe(self):
        if self.loss[0] == "ge":
            kind = "GE loss (p_gb=0.0155,p_bg=0.5) on body shards"
        elif self.loss[0] == "bern":
            kind = "Bernoulli %.0f%% body-shard loss" % (100 * self.loss[1])
        else:
            kind = "%.0f%% synthetic block mask (data.synthetic_mask)" % (100 * self.loss[1])
        mod = "RGB + 16-bit depth" if self.depth16 else "RGB-D"
        return "%dx%d %s, %d streams, %s" % (self.w, self.h, mod, len(self.ids), kind)


class ModalityWork:
    """The streams of one modality of a Workload on one GPU: device-resident
    reference planes + corrupted planes, loss-mask jobs (or block masks),
    pinned host copies, the engine, and (headline) the serving pipeline."""

    def __init__(self, wl: Workload, name, c, L, device, precision, pipeline=False, engine=None):
        from paper_2604_27441_b200 import Checkpoint, ModelConfig
        from paper_2604_27441_b200.lossmask import LossMaskBatch, PFrameShards
        from paper_2604_27441_b200.recovery import RecoveryEngine, pack_grid, stack_slots

        h, w = wl.h, wl.w
        S = len(wl.ids)
        self.name, self.c, self.S, self.h, self.w = name, c, S, h, w
        cfg = ModelConfig()
        if engine is None:
            ck = Checkpoint.random_init(cfg, c, seed=0)          # torch.manual_seed(0) init
            engine = RecoveryEngine(ck.build_model(precision=precision), precision)
        self.engine = engine
        self.engine.model.native(device)
        F = cfg.stack_len
        # 16-bit depth: u16 (h, w) planes through nvrec_recover_u16
        self.u16 = bool(wl.depth16 and c == 1)
        shape = (h, w) if self.u16 else (h, w, c)
        dt = torch.uint16 if self.u16 else torch.uint8
        self.host_frames = torch.empty((S * F,) + shape, dtype=dt).pin_memory()
        hf = self.host_frames.numpy().reshape((S, F) + shape)
        for s, sid in enumerate(wl.ids):
            hf[s] = stream_planes16(h, w, sid) if self.u16 else wl.planes(c, sid)
        self.frames = self.host_frames.to(device)
        self.ring_view = self.frames.view((S, F) + shape)
        self.host_planes = self.host_frames.view((S, F) + shape)[:, -1].contiguous().pin_memory()
        self.recover = engine.recover_device16 if self.u16 else engine.recover_device
        self.index = torch.tensor([[s * F + i for i in stack_slots(5, 5, F)]
                                   for s in range(S)], dtype=torch.int32, device=device)
        nblk = (h // 16) * (w // 16)
        self.jobs, self.lm = None, None
        if wl.loss[0] in ("ge", "bern"):
            self.jobs = []
            for s, sid in enumerate(wl.ids):
                hdr, nd, recv, enc = wl.job(c, L, s, sid)
                self.jobs.append(PFrameShards(hdr, nd, recv, L, enc))
            self.lm = LossMaskBatch(S, max(len(j.header) for j in self.jobs) + 16,
                                    max(j.n_data for j in self.jobs) + 1, nblk, 1, device)
            self.lm.stage(self.jobs)
            self.lm.launch()
            grids = self.lm.results()
            self.wire = self.lm.wire
        else:
            grids = [wl.grid(c, sid) for sid in wl.ids]
            bits = np.stack([pack_grid(g) for g in grids])
            self.host_wire = torch.from_numpy(bits).pin_memory()
            self.wire = self.host_wire.to(device)
        self.masked_patches = [int(g.sum()) for g in grids]
        self.out = torch.empty((S,) + shape, dtype=dt, device=device)
        self.host_out = torch.empty((S,) + shape, dtype=dt).pin_memory()
        self.pipe = None
        if pipeline and self.jobs is not None:
            from paper_2604_27441_b200.recovery import RecoveryPipeline
            self.pipe = RecoveryPipeline(self.engine, S, h, w, L, self.lm.max_header,
                                         self.lm.max_shards, self.ring_view[:, :cfg.k])
            for buf in self.pipe.host_in:
                buf.copy_(self.host_planes)           # the decoder writes planes here

    def _mask(self, stream):
        from paper_2604_27441_b200 import _native
        import ctypes
        if self.lm is not None:
            _native.check(self.lm.lib.nvrec_loss_mask(ctypes.c_void_p(self.lm.dev_in.data_ptr()),
                                                      self.lm.n,
                                                      ctypes.c_void_p(int(stream.cuda_stream))))

    def device_step(self, stream):
        """Loss mask + recovery with inputs resident in HBM, merged in place
        (the serving mode of RecoveryPipeline: the recovered patches land in
        the corrupted plane's slot; the model never reads those pixels, so
        repeating the step recomputes the same plane)."""
        self._mask(stream)
        self.recover(self.frames, self.index, self.wire, in_place=True)

    def e2e_step(self, stream):
        """Unpipelined end to end: H2D of each stream's corrupted plane and
        its loss-mask job (or mask bits), recovery against the device-resident
        references, ring push (D2D), D2H of the recovered planes."""
        if self.lm is not None:
            self.lm.launch(stream)                           # H2D jobs + kernel
        else:
            self.wire.copy_(self.host_wire, non_blocking=True)
        self.ring_view[:, -1].copy_(self.host_planes, non_blocking=True)
        self.recover(self.frames, self.index, self.wire, self.out)
        self.ring_view[:, -2].copy_(self.out, non_blocking=True)   # ring push
        self.host_out.copy_(self.out, non_blocking=True)

    def protocol_step(self, stream):
        """Reference wire-protocol semantics (recovery.py:219-227): every
        request ships the corrupted plane AND all k references (H2D)."""
        self.lm.launch(stream)
        self.frames.copy_(self.host_frames, non_blocking=True)
        self.engine.recover_device(self.frames, self.index, self.wire, self.out)
        self.host_out.copy_(self.out, non_blocking=True)

    def h2d_bytes(self):
        m = self.lm.h2d_bytes if self.lm is not None else self.host_wire.numel()
        return int(m + self.host_planes.numel() * self.host_planes.element_size())

    def h2d_bytes_protocol(self):
        return int(self.lm.h2d_bytes + self.host_frames.numel())

    def d2h_bytes(self):
        return int(self.host_out.numel() * self.host_out.element_size())


class ReceiverWork:
    """S streams of one modality as the receiver sees them: per frame time a
    codec P-frame (synthetic talking-motion content, encoded by the sender
    restatement in tools/synth.py) whose body shards went through the GE
    channel; decoded + recovered on the GPU by ReceiverPipeline."""

    def __init__(self, name, c, L, stream_ids, device, engine, n_frames=6):
        from tools import synth
        from paper_2604_27441_b200.receiver import ReceiverPipeline
        from tools.synth import GilbertElliott
        self.name, self.c, self.S = name, c, len(stream_ids)
        seqs, init = [], []
        max_hdr = max_body = max_nd = 0
        for s, sid in enumerate(stream_ids):
            clip = synth.talking_clip(n_frames + 1, W, H, c, seed=sid * 7 + c)
            seq = []
            ge = GilbertElliott(seed=sid + 31 * c)
            prev = clip[0]                        # sender reference (lossless side)
            for f in clip[1:]:
                hp, pp = synth.encode_p(f, prev)
                nd = synth.n_data_shards(len(pp), L)
                recv = np.ones(nd, bool)
                for i in range(1, nd):
                    recv[i] = not ge.drop()
                if recv.all():
                    recv[1 + (s % max(1, nd - 1))] = False
                seq.append((hp, synth.receiver_body(pp, L, recv), recv, L))
                max_hdr, max_body, max_nd = max(max_hdr, len(hp)), max(max_body, len(pp)), \
                    max(max_nd, nd)
                prev = f
            seqs.append(seq)
            init.append(np.stack([clip[0]] * 5).reshape(5, H, W, c))
        self.seqs = seqs
        self.n_frames = n_frames
        init_t = torch.from_numpy(np.stack(init)).to(device)
        self.pipe = ReceiverPipeline(engine, self.S, H, W, init_t, max_hdr + 16, max_body + 16,
                                     max_nd + 1)
        self.t = 0

    def submit(self):
        j = self.t % self.n_frames
        self.t += 1
        return self.pipe.submit([seq[j] for seq in self.seqs])


def _events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed_receiver(rworks, steps, dist_on):
    """Receiver back end end to end: compressed P-frames in (pinned H2D),
    GPU decode + loss mask + recovery, displayable planes out (D2H)."""
    main = torch.cuda.current_stream()
    torch.cuda.synchronize()
    if dist_on:
        torch.distributed.barrier()
    t0, t1 = _events()
    t0.record(main)
    for rw in rworks:
        rw.pipe.s_h2d.wait_event(t0)
    h2d = 0
    for _ in range(steps):
        for rw in rworks:
            hnd = rw.submit()
            h2d += rw.pipe.h2d_bytes(hnd)
    for rw in rworks:
        main.wait_stream(rw.pipe.s_d2h)
    t1.record(main)
    torch.cuda.synchronize()
    return max_over_ranks(t0.elapsed_time(t1), dist_on, "cuda"), h2d / steps


def timed_pipeline(works, steps, dist_on):
    """End-to-end serving throughput: every step submits each stream's new
    corrupted plane + loss-mask job from pinned host memory and returns the
    recovered planes to the host (RecoveryPipeline: H2D, compute and D2H of
    consecutive steps overlap).  Device-timed from the first H2D to the last
    D2H with CUDA events on a stream all pipeline streams are ordered after."""
    main = torch.cuda.current_stream()
    torch.cuda.synchronize()
    if dist_on:
        torch.distributed.barrier()
    t0, t1 = _events()
    t0.record(main)
    for wk in works:
        wk.pipe.s_h2d.wait_event(t0)
    for _ in range(steps):
        for wk in works:
            wk.pipe.submit(None, wk.jobs)
    for wk in works:
        main.wait_stream(wk.pipe.s_d2h)
    t1.record(main)
    torch.cuda.synchronize()
    return max_over_ranks(t0.elapsed_time(t1), dist_on, "cuda")


def run_steps(works, streams, fn, n, join_each_step=True):
    """n steps of every modality on its own stream.  join_each_step: all
    modalities finish step t before any starts t+1 (a frame-time barrier);
    otherwise each modality stream runs its steps back to back (in order, so
    a step still follows the one whose output it would take as a reference)
    and the streams join once at the end -- what a server does, and what the
    e2e pipelines measure."""
    main = torch.cuda.current_stream()
    ev = main.record_event()
    for st in streams:
        st.wait_event(ev)
    for _ in range(n):
        if join_each_step:
            ev = main.record_event()
            for st in streams:
                st.wait_event(ev)
        for wk, st in zip(works, streams):
            with torch.cuda.stream(st):
                getattr(wk, fn)(st)
        if join_each_step:
            for st in streams:
                main.wait_stream(st)
    for st in streams:
        main.wait_stream(st)


def timed(works, streams, fn, steps, dist_on, join_each_step=True):
    torch.cuda.synchronize()
    if dist_on:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0, t1 = _events()
    t0.record()
    run_steps(works, streams, fn, steps, join_each_step)
    t1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(t0.elapsed_time(t1), dist_on, "cuda")
    if dist_on:
        torch.distributed.barrier()
    return ms


# ----------------------------------------------------------------------------
# algorithmic work for the roofline of the dominant kernel

def attention_flops(ns, n_masked, nt=3, heads=2, hd=32, layers=2):
    """Spatial attention FLOPs actually required per modality-frame:
    dense blocks need all ns queries; the last block only the masked ones
    (exact pruning, the merge discards the rest)."""
    per_q = 4 * ns * hd * heads * nt          # QK^T + PV per query row
    return per_q * (ns * (layers - 1) + n_masked)


# ----------------------------------------------------------------------------
# reference CPU path (the oracle restatement; test infrastructure)

class CpuReference:
    """The reference CPU path on a Workload's inputs: per stream-frame and
    modality, the receiver/codec loss mask (oracle.lossmask, restating
    receiver.py:224-237 + codec.py:250-281) and RecoveryServer._recover
    (oracle.recover, server.py:181-196) in fp32 torch-CPU, with the same
    random-init weights (seed 0) and planes as the GPU arm."""

    def __init__(self, wl: Workload, threads=None):
        from oracle import nvrec_forward, recover as orec, lossmask as olm
        from paper_2604_27441_b200.checkpoint import Checkpoint
        from paper_2604_27441_b200.config import ModelConfig
        self.threads = threads or (os.cpu_count() or 1)
        torch.set_num_threads(self.threads)
        self.arch = nvrec_forward.Arch()
        self.orec, self.olm, self.wl = orec, olm, wl
        self.states, self.inputs = {}, {}
        for name, c, L in MODS:
            ck = Checkpoint.random_init(ModelConfig(), c, seed=0)
            self.states[c] = {k: v.numpy() for k, v in ck.state.items()}
            per = []
            for s, sid in enumerate(wl.ids):
                fr = wl.planes(c, sid)
                per.append((fr, wl.job(c, L, s, sid) if wl.loss[0] != "block" else wl.grid(c, sid), L))
            self.inputs[c] = per
        self.i = 0

    def frame(self):
        """One stream's RGB-D frame (both modalities), round robin."""
        s = self.i % len(self.wl.ids)
        self.i += 1
        for _, c, _ in MODS:
            fr, m, L = self.inputs[c][s]
            if isinstance(m, tuple):
                hdr, nd, recv, enc = m
                grid = self.olm.mask_from_shards(hdr, nd, set(np.flatnonzero(recv).tolist()), L, enc)
            else:
                grid = m
            self.orec.recover(self.states[c], self.arch, c, fr[-1], grid, list(fr[:-1]))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference(wl, seconds, threads=None, max_frames=None):
    """Frames/s of the reference CPU path over a bounded sample."""
    ref = CpuReference(wl, threads)
    ref.frame()                               # warm-up
    n, t0 = 0, time.perf_counter()
    while True:
        ref.frame()
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or (max_frames and n >= max_frames):
            break
    return n / el, n, el, ref.threads


def headline_workload(streams_total: int) -> Workload:
    return Workload("720p_ge", H, W, range(streams_total), ("ge",))


def reference_arm(args, rank, world):
    if rank != 0:
        return
    wl = headline_workload(args.streams_per_gpu * world)
    ref = CpuReference(wl)
    for _ in range(args.warmup):
        ref.frame()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.frame()
    tot = time.perf_counter() - t0
    threads = ref.threads
    value = args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD_720P % args.streams_per_gpu,
                       "streams_per_gpu": args.streams_per_gpu, "height": H, "width": W,
                       "same_inputs_as_gpu_arm": True,
                       "sample": "each step = one stream's RGB-D frame (round robin over the "
                                 "%d streams): the same planes, GE-dropped shards and weights "
                                 "as the GPU arm's step" % (args.streams_per_gpu * world)},
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads,
                             "kind": "port", "cpu_model": cpu_model(),
                             "sample": "%d x 720p RGB-D stream-frames through the oracle "
                                       "restatement of the receiver loss mask + "
                                       "RecoveryServer._recover (fp32 torch-CPU, %d threads)"
                                       % (args.steps, threads)},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def dry_run(args, rank, world):
    """Launch / timing / reporting logic without a GPU (CPU tests)."""
    dist_on = world > 1
    if dist_on:
        torch.distributed.init_process_group("gloo")
    t0 = time.perf_counter()
    x = torch.ones(1 << 16)
    for _ in range(args.steps):
        x = x * 1.0001
    ms = max_over_ranks(1000 * (time.perf_counter() - t0), dist_on)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms / max(1, args.steps),
                          "streams_total": args.streams_per_gpu * world,
                          "scaling": "weak"}), flush=True)
    if dist_on:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


# ----------------------------------------------------------------------------
# our arm

def measure_config(wl, device, precision, steps, warmup, dist_on, engines=None):
    """Device-resident throughput + unpipelined e2e of one extra config."""
    works = [ModalityWork(wl, n, c, L, device, precision,
                          engine=engines[i] if engines else None)
             for i, (n, c, L) in enumerate(MODS)]
    streams = [torch.cuda.Stream(device) for _ in works]
    run_steps(works, streams, "device_step", warmup)
    ms = timed(works, streams, "device_step", steps, dist_on, join_each_step=False)
    run_steps(works, streams, "e2e_step", 2)
    ms_e2e = timed(works, streams, "e2e_step", steps, dist_on)
    n = len(wl.ids) * steps
    out = {"workload": wl.describe(), "value": n / (ms / 1e3),
           "e2e_unpipelined": n / (ms_e2e / 1e3), "unit": "frames/s",
           "ms_per_step": ms / steps,
           "masked_patches_per_frame": {wk.name: float(np.mean(wk.masked_patches)) for wk in works},
           "h2d_bytes_per_step": sum(wk.h2d_bytes() for wk in works),
           "d2h_bytes_per_step": sum(wk.d2h_bytes() for wk in works)}
    del works
    torch.cuda.empty_cache()
    return out


def measure_module_api(engines, device, h, w, streams, steps):
    """The float drop-in (reference model.py:82-122 signature): dense forward
    of every patch of ``streams`` RGB-D float stacks, inputs resident."""
    out = {}
    for eng, (name, c, _) in zip(engines, MODS):
        model = eng.model
        g = torch.Generator(device="cpu").manual_seed(5)
        stack = torch.rand(streams, 6, c, h, w, generator=g).to(device)
        mask = (torch.rand(streams, h, w, generator=g) < 0.1).to(device)
        for _ in range(2):
            model(stack, mask)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            model(stack, mask)
        e1.record()
        torch.cuda.synchronize()
        out[name + "_ms_per_call"] = e0.elapsed_time(e1) / steps
    ms = sum(v for v in out.values())
    out.update({"value": streams / (ms / 1e3), "unit": "frames/s",
                "note": "RGB + depth module calls back to back, precision as the headline; "
                        "the float path embeds on CUDA cores (embed_kernel + ln_qkv_kernel), "
                        "every later stage on the tensor-core kernels"})
    return out


def main():
    args = parse()
    spawn_ranks(args)
    rank, world, local = dist_env()
    dist_on = world > 1
    if args.dry_run:
        dry_run(args, rank, world)
        return
    if args.impl == "reference":
        if dist_on:
            torch.distributed.init_process_group("gloo")
        reference_arm(args, rank, world)
        if dist_on:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return
    from paper_2604_27441_b200 import _native
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if dist_on:
        torch.distributed.init_process_group("nccl", device_id=device)
    S = args.streams_per_gpu
    from paper_2604_27441_b200.sharding import streams_for_rank
    mine = streams_for_rank(S * world, rank, world)       # stream s -> GPU s mod N
    wl = Workload("720p_ge", H, W, mine, ("ge",))
    works = [ModalityWork(wl, n, c, L, device, args.precision, pipeline=True)
             for n, c, L in MODS]
    streams = [torch.cuda.Stream(device) for _ in works]

    # warm-up (both paths), then the device-resident timed region
    run_steps(works, streams, "device_step", args.warmup)
    run_steps(works, streams, "e2e_step", max(1, args.warmup // 2))
    # device throughput: modality streams run their steps back to back (the
    # e2e pipelines overlap the same way); the per-step-barrier figure is
    # reported beside it
    with ClockSampler(local) as clocks:
        ms = timed(works, streams, "device_step", args.steps, dist_on, join_each_step=False)
    clk = clocks.result()
    ms_joined = timed(works, streams, "device_step", args.steps, dist_on)
    # end-to-end through host buffers (streaming backend) and the reference
    # wire-protocol variant that re-ships all k references every request
    for wk in works:                                         # pipeline warm-up
        for _ in range(3):
            wk.pipe.submit(None, wk.jobs)
    torch.cuda.synchronize()
    ms_e2e = timed_pipeline(works, args.steps, dist_on)
    ms_e2e_serial = timed(works, streams, "e2e_step", max(3, args.steps // 4), dist_on)
    ms_proto = timed(works, streams, "protocol_step", max(3, args.steps // 4), dist_on)
    # receiver back end: compressed P-frames in, decode + recovery on the GPU
    rworks = [ReceiverWork(n, c, L, mine, device, wk.engine) for (n, c, L), wk in zip(MODS, works)]
    for _ in range(4):
        for rw in rworks:
            rw.submit()
    torch.cuda.synchronize()
    ms_recv, recv_h2d = timed_receiver(rworks, args.steps, dist_on)
    del rworks
    # per-stage device times: separate pass, both modalities serialised on ONE
    # stream so event brackets are not inflated by the concurrent modality
    torch.cuda.synchronize()
    one = [torch.cuda.current_stream(device)] * len(works)
    with _native.StageProfile() as prof:
        run_steps(works, one, "device_step", args.steps)
        torch.cuda.synchronize()

    # single-stream RGB-D latency (b = 1 per modality, e2e through host buffers)
    lat = []
    if rank == 0:
        single_wl = Workload("720p_single", H, W, [999], ("ge",))
        single = [ModalityWork(single_wl, n, c, L, device, args.precision)
                  for n, c, L in MODS]
        sst = [torch.cuda.Stream(device) for _ in single]
        run_steps(single, sst, "e2e_step", 5)
        for _ in range(args.latency_iters):
            lat.append(timed(single, sst, "e2e_step", 1, False))
        lat_dev = [timed(single, sst, "device_step", 1, False)
                   for _ in range(args.latency_iters)]
        lat_proto = [timed(single, sst, "protocol_step", 1, False)
                     for _ in range(args.latency_iters)]
        del single

    # the other BASELINE configs and densities (device value + unpipelined e2e)
    extra, fast = {}, None
    if not args.no_extra:
        k = max(5, args.steps // 10)
        other = "fast" if args.precision == "precise" else "precise"
        # the other precision on the headline workload
        wk2 = [ModalityWork(wl, n, c, L, device, other, pipeline=True) for n, c, L in MODS]
        st2 = [torch.cuda.Stream(device) for _ in wk2]
        run_steps(wk2, st2, "device_step", args.warmup)
        ms2 = timed(wk2, st2, "device_step", args.steps, dist_on, join_each_step=False)
        for wk in wk2:
            for _ in range(3):
                wk.pipe.submit(None, wk.jobs)
        torch.cuda.synchronize()
        ms2_e2e = timed_pipeline(wk2, args.steps, dist_on)
        n2 = S * world * args.steps
        fast = {"precision": other, "dtype": "bf16" if other == "fast" else PRECISE_DTYPE,
                "value": n2 / (ms2 / 1e3), "unit": "frames/s", "ms_per_step": ms2 / args.steps,
                "e2e": {"value": n2 / (ms2_e2e / 1e3), "unit": "frames/s",
                        "h2d_bytes_per_step": sum(w.pipe.h2d_bytes() for w in wk2),
                        "d2h_bytes_per_step": sum(w.pipe.d2h_bytes() for w in wk2)},
                "note": "same workload and timing as the headline, %s operands" %
                        ("bf16/fp16 tensor-core (max-abs 2.6e-4 at 720p)" if other == "fast"
                         else "split (fp32-class)")}
        del wk2
        torch.cuda.empty_cache()
        engines = [w.engine for w in works]
        cfgs = [
            ("configs[0] 320x240 10% block", Workload("c0", 240, 320, mine, ("block", 0.10))),
            ("configs[1] 640x480 Bernoulli 5%", Workload("c1", 480, 640, mine, ("bern", 0.05))),
            ("configs[1] 640x480 RGB + 16-bit depth, Bernoulli 5%",
             Workload("c1d16", 480, 640, mine, ("bern", 0.05), depth16=True)),
            ("configs[2] 720p 10% block", Workload("c2b10", H, W, mine, ("block", 0.10))),
            ("configs[2] 720p 20% block", Workload("c2b20", H, W, mine, ("block", 0.20))),
            ("configs[3] 1920x1088 20% block", Workload("c3", 1088, 1920, mine, ("block", 0.20))),
            ("configs[4] 64 streams x 720p GE on this GPU",
             Workload("c4", H, W, streams_for_rank(64, rank, world), ("ge",))),
        ]
        for key, cwl in cfgs:
            extra[key] = measure_config(cwl, device, args.precision, k, 2, dist_on, engines)
        extra["module API MaskedVideoModel.forward 8 x 720p (dense, float stacks)"] = \
            measure_module_api(engines, device, H, W, S, k)

    if dist_on:
        torch.distributed.barrier()
    if rank != 0:
        torch.distributed.destroy_process_group()
        return

    frames = S * world * args.steps
    value = frames / (ms / 1000.0)
    e2e = frames / (ms_e2e / 1000.0)
    # roofline of the dominant kernel (spatial attention)
    ns = (H // 16) * (W // 16)
    att_kind = "attn_tc" if prof.launches["attn_tc"] else "attn_simt"
    att_ms = prof.ms[att_kind]
    att_launches = prof.launches[att_kind]
    flops = 0
    for wk in works:
        for m in wk.masked_patches:
            flops += attention_flops(ns, m)
    flops *= args.steps
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peaks = json.load(open(peaks_path))
        peak, peak_src = peaks["bf16_tflops"], "MEASURED_PEAKS.json bf16_tflops (burst)"
    else:
        peak, peak_src = 1590.0, "fallback B200_PROFILING.md"
    achieved = flops / (att_ms / 1000.0) / 1e12 if att_ms else 0.0
    exps = flops / 128.0                      # 4*hd = 128 MMA-FLOP per score
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "attn_tc_ncu.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath)).get(args.precision, {})
        traffic = tj.get("dram_bytes_per_launch")
        traffic_src = tj.get("source")
    launches_per_step = prof.total_launches / args.steps
    precise = args.precision == "precise"
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "value_frame_barrier": frames / (ms_joined / 1000.0),
        "value_note": "value: each modality stream runs its steps back to back and the "
                      "streams join at the end (as the e2e pipelines run); "
                      "value_frame_barrier: both modalities finish step t before t+1 starts",
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": PRECISE_DTYPE if precise else "bf16",
        "precision": PRECISE_NOTE if precise else "fast: bf16/fp16 tensor-core operands, fp32 "
                                                  "accumulation (720p max-abs 2.6e-4)",
        "data": "synthetic",
        "config": {"workload": WORKLOAD_720P % S,
                   "streams_per_gpu": S, "height": H, "width": W,
                   "precision": args.precision,
                   "same_inputs_as_reference_arm": True,
                   "masked_patches_per_frame": {wk.name: float(np.mean(wk.masked_patches))
                                                for wk in works},
                   "l2": "inputs larger than L2 (%.0f MB of u8 planes per step > 126 MB)"
                         % (sum(wk.host_frames.numel() for wk in works) / 1e6)},
        "clocks": clk,
        "e2e": {"value": e2e, "unit": "frames/s",
                "h2d_bytes_per_step": sum(wk.pipe.h2d_bytes() for wk in works),
                "d2h_bytes_per_step": sum(wk.pipe.d2h_bytes() for wk in works),
                "path": "RecoveryPipeline (public serving API): per step pinned H2D of each "
                        "stream's corrupted plane + loss-mask job + slot table, loss-mask "
                        "kernel, recovery on device-resident k=5 reference rings, ring push, "
                        "D2H of the recovered planes; consecutive steps double-buffered so "
                        "copies overlap compute"},
        "e2e_unpipelined": {"value": S * world * max(3, args.steps // 4) / (ms_e2e_serial / 1000.0),
                            "unit": "frames/s",
                            "path": "same transfers, H2D -> compute -> D2H serialised per step"},
        "e2e_protocol": {"value": S * world * max(3, args.steps // 4) / (ms_proto / 1000.0),
                         "unit": "frames/s",
                         "h2d_bytes_per_step": sum(wk.h2d_bytes_protocol() for wk in works),
                         "d2h_bytes_per_step": sum(wk.d2h_bytes() for wk in works),
                         "path": "reference wire-protocol payload: all k references re-sent "
                                 "per request (recovery.py:219-227)"},
        "e2e_receiver": {"value": S * world * args.steps / (ms_recv / 1000.0), "unit": "frames/s",
                         "h2d_bytes_per_step": int(recv_h2d),
                         "d2h_bytes_per_step": sum(wk.d2h_bytes() for wk in works),
                         "path": "ReceiverPipeline: per step each stream's received P-frame "
                                 "(codec header + assembled body with zero-filled lost "
                                 "shards, receiver.py:222-237) H2D, nvrec_decode (zero-fill "
                                 "decode + loss mask, codec.py:260-321) against the newest "
                                 "ring plane, nvrec_recover_u8 into the ring, D2H of the "
                                 "displayable planes; synthetic talking-motion 720p content "
                                 "encoded by the tools/synth.py sender, GE channel loss"},
        "gpu_launches": int(round(launches_per_step * args.steps)),
        "p50_latency_ms": statistics.median(lat),
        "p99_latency_ms": float(np.percentile(lat, 99)),
        "p50_latency_device_ms": statistics.median(lat_dev),
        "p50_latency_protocol_ms": statistics.median(lat_proto),
        "latency_note": "single stream, one RGB-D frame (both modalities on two CUDA "
                        "streams), e2e through pinned host buffers incl. H2D of the "
                        "corrupted plane + loss-mask job per modality (references device-"
                        "resident) and D2H of the result; _device = inputs resident; "
                        "_protocol = all 6 planes per modality shipped as the reference "
                        "wire protocol does",
        "stage_ms_per_step": {k: v / args.steps for k, v in prof.ms.items() if v},
        "stage_note": "per-stage device ms from CUDA-event brackets, both modalities "
                      "serialised on one stream (separate pass)",
        "roofline": {"kernel": att_kind + (" (split-bf16 x3)" if precise else ""),
                     "bound": "tensor", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "binding_unit": "mufu (SFU ex2): head_dim 32 gives 128 MMA-FLOP per "
                                     "exponential, so the exp rate, not the tensor core, "
                                     "bounds this kernel; see roofline.mufu.frac",
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src,
                     "mufu": {"exp_per_s": exps / (att_ms / 1000.0) if att_ms else 0.0,
                              "peak_exp_per_s": MUFU_PEAK,
                              "frac": (exps / (att_ms / 1000.0) / MUFU_PEAK) if att_ms else 0.0,
                              "note": "binding unit for head_dim 32 (128 MMA-FLOP per exp); "
                                      "peak = 148 SM x 16 ex2/clk x 1.965 GHz (15.9 ex2/clk/SM "
                                      "measured by tools/ubench_xu.cu); " +
                                      ("all exps on MUFU (fp32-accurate ex2.approx)" if precise
                                       else "1/4 of the exps run as FMA-pipe polynomials")},
                     "algorithmic_note": "achieved counts the reference-equivalent (pruned) "
                                         "attention FLOPs, not the 3x MMA work of the split "
                                         "products" if precise else "reference-equivalent "
                                         "(pruned) attention FLOPs",
                     "share_of_step": att_ms / max(1e-9, sum(prof.ms.values())),
                     "algorithmic_flops_per_launch": flops / max(1, att_launches)},
    }
    if fast is not None:
        line["other_precision"] = fast
    if extra:
        line["configs"] = extra
    if not args.no_cpu_baseline:
        fps, n, el, threads = cpu_reference(wl, args.cpu_seconds)
        fps1, n1, el1, _ = cpu_reference(wl, min(6.0, args.cpu_seconds / 2), threads=1,
                                         max_frames=3)
        torch.set_num_threads(os.cpu_count() or 1)
        line["cpu_baseline"] = {"value": fps, "unit": "frames/s", "cores": threads,
                                "kind": "port", "cpu_model": cpu_model(),
                                "sample": "%d x 720p RGB-D stream-frames of the headline "
                                          "workload (%.1f s) through the oracle restatement of "
                                          "the receiver loss mask + RecoveryServer._recover, "
                                          "fp32 torch-CPU, %d threads" % (n, el, threads),
                                "threads_1": {"value": fps1, "unit": "frames/s", "cores": 1,
                                              "sample": "%d stream-frames (%.1f s)" % (n1, el1)}}
    print(json.dumps(line), flush=True)
    if dist_on:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
