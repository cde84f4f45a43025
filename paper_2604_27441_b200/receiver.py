"""Device-resident receiver back end: P-frame decode + recovery on the GPU.

Replaces, for ``n`` streams of one modality, the tail of the reference
receiver's P-frame finalisation (rgbdstream/receiver.py:211-274):

  body assembly      received body shards + zero chunks (receiver.py:228-237)
                     -- done by the caller on the host, it is what arrived
  codec.decode       zero-fill decode against the stream's newest displayable
                     plane (``self.refs[modality]``, receiver.py:244-247) and
                     the corruption mask (codec.py:260-321) -> nvrec_decode
  backend(req)       recovery with the k-frame ring (receiver.py:260-264)
                     -> nvrec_recover_u8 in place: the masked patches are
                     written into the decoded plane's own slot
  ring push          that slot becomes the newest reference and the oldest
                     leaves the ring (receiver.py:268-269) -- a cyclic slot
                     schedule, no copies

Per frame time only the compressed bytes travel host -> device (codec header
+ assembled body, ~60-200 KB at 720p instead of a 2.8 MB plane), and the
displayable plane comes back.  Decode errors (``UndecodableError`` in the
reference, i.e. LOST_FRAME, receiver.py:244-248) are reported per stream by
``result``.  The reference then displays nothing and leaves its references
alone; here every stream's ring advances together, so the lost frame's slot
receives a copy of the newest displayable plane (the next P-frame decodes
against the same plane as in the reference) and recovers nothing (its wire
bits are cleared on the device).  The one deviation: the ring holds the
newest plane twice instead of keeping its oldest reference for one more
frame.
"""

from __future__ import annotations

import torch

from . import _native
from .codec import DecodeBatch, DecodeItem, raise_status
from .recovery import RecoveryEngine, cyclic_slot_tables


class ReceiverPipeline:
    """Pipelined receive -> decode -> recover loop for ``n`` streams.

    ``submit(frames)`` takes one received P-frame per stream as
    (header bytes, assembled body bytes, received-shard flags, shard_len) and
    returns a handle; ``result(handle)`` returns the displayable planes
    (n, h, w, c) in pinned host memory and the per-stream decode status."""

    def __init__(self, engine: RecoveryEngine, n: int, h: int, w: int, init_refs: torch.Tensor,
                 max_header: int, max_payload: int, max_shards: int, nbuf: int = 3,
                 graphs: bool = True):
        self.engine = engine
        self.n, self.h, self.w = n, h, w
        self.c = engine.channels
        cfg = engine.model.config
        self.k, self.F = cfg.k, cfg.stack_len
        self.nbuf = nbuf
        dev = init_refs.device
        self.device = dev
        # S = k + nbuf slots used cyclically (see RecoveryPipeline): step t
        # decodes into slot t+k against the newest reference t+k-1
        self.S = self.k + nbuf
        self.frames = torch.empty((self.S, n, h, w, self.c), dtype=torch.uint8, device=dev)
        self.frames[:self.k].copy_(init_refs.transpose(0, 1))      # (n, k, ...) -> slot-major
        self.flat = self.frames.view(self.S * n, h, w, self.c)
        nblk = (h // 16) * (w // 16)
        self.dec = [DecodeBatch(n, max_header, max_payload, nblk, max_shards=max_shards,
                                max_ranges=1, device=dev) for _ in range(nbuf)]
        self.host_out = [torch.empty((n, h, w, self.c), dtype=torch.uint8).pin_memory()
                         for _ in range(nbuf)]
        self.tables = cyclic_slot_tables(self.k, nbuf, n, self.F, dev)
        # the step's slot table rides in with its inputs, so one CUDA graph
        # (decode + recovery) per buffer set serves every ring phase
        self.tab_cur = torch.empty((nbuf, n, self.F), dtype=torch.int32, device=dev)
        self.nat = engine.model.native_snapshot(dev)  # private weight snapshot
        self.use_graphs = graphs
        self._graphs = {}
        self.s_h2d = torch.cuda.Stream(dev)
        self.s_cmp = torch.cuda.Stream(dev)
        self.s_d2h = torch.cuda.Stream(dev)
        self.ev_h2d = [torch.cuda.Event() for _ in range(nbuf)]
        self.ev_cmp = [torch.cuda.Event() for _ in range(nbuf)]
        self.ev_d2h = [torch.cuda.Event() for _ in range(nbuf)]
        self.step = 0
        self.bytes_in = [0] * nbuf

    def h2d_bytes(self, handle: int | None = None) -> int:
        """Compressed bytes shipped for one step (headers + bodies + descriptors)."""
        return int(self.bytes_in[self.step % self.nbuf if handle is None else handle])

    def d2h_bytes(self) -> int:
        return int(self.host_out[0].numel())

    def submit(self, frames) -> int:
        """frames: n tuples (header, body, received flags, shard_len)."""
        i = self.step % self.nbuf
        if self.step >= self.nbuf:
            self.ev_h2d[i].synchronize()
            self.ev_d2h[i].synchronize()
        ph = self.step % self.S
        st = (self.step + self.k) % self.S              # decoded plane's slot
        newest = (st - 1) % self.S
        items = []
        for s, (header, body, received, shard_len) in enumerate(frames):
            items.append(DecodeItem(header, body, self.frames[st, s],
                                    self.frames[newest, s], n_data=len(received),
                                    received=received, shard_len=shard_len,
                                    body_len=len(body)))
        dec = self.dec[i]
        dec.stage(items)
        self.bytes_in[i] = dec.used
        if self.step >= self.nbuf:
            self.s_h2d.wait_event(self.ev_cmp[i])       # staging buffer of step - nbuf read
        with torch.cuda.stream(self.s_h2d):
            # descriptors, headers, flags and the packed bodies: one copy
            dec.dev_in[:dec.used].copy_(dec.host[:dec.used], non_blocking=True)
            self.tab_cur[i].copy_(self.tables[ph], non_blocking=True)
            self.ev_h2d[i].record(self.s_h2d)
        # decode into slot st (last read by step - nbuf's compute, earlier on
        # s_cmp), then recover in place: st becomes the newest reference
        self.s_cmp.wait_event(self.ev_h2d[i])
        self._run(i)
        self.ev_cmp[i].record(self.s_cmp)
        self.s_d2h.wait_event(self.ev_cmp[i])
        with torch.cuda.stream(self.s_d2h):
            self.host_out[i].copy_(self.frames[st], non_blocking=True)
            self.ev_d2h[i].record(self.s_d2h)
        self.step += 1
        return i

    def _compute(self, i: int) -> None:
        dec = self.dec[i]
        with torch.cuda.stream(self.s_cmp):
            dec.launch(self.s_cmp, copy=False)
            self.engine.recover_device(self.flat, self.tab_cur[i], dec.wire, in_place=True,
                                       native=self.nat)

    def _run(self, i: int) -> None:
        if not self.use_graphs:
            self._compute(i)
            return
        g = self._graphs.get(i)
        if g is None:
            # first use: run eagerly (warms attributes and the workspace), then
            # capture for the following steps of this buffer set
            self._compute(i)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.s_cmp):
                self._compute(i)
            self._graphs[i] = g
            return
        with torch.cuda.stream(self.s_cmp):
            g.replay()

    def result(self, handle: int, check: bool = True):
        """(planes (n, h, w, c), per-stream decode status codes).  With
        ``check`` the first failing stream raises like ``codec.decode``."""
        self.ev_d2h[handle].synchronize()
        st = self.dec[handle].status[:self.n, 0].cpu().numpy()
        if check:
            for s in range(self.n):
                raise_status(int(st[s]), self.dec[handle].headers[s])
        return self.host_out[handle].numpy(), st
