"""World-size-2 gloo run of the stream-sharding host logic (CPU): every
stream has exactly one owner, routing keeps per-stream order, and the
benchmark's max-over-ranks timing reduction works without a GPU."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_27441_b200.sharding import owner, route, streams_for_rank


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_streams, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = streams_for_rank(n_streams, rank, world)
    ids = torch.full((n_streams,), -1, dtype=torch.int64)
    ids[:len(mine)] = torch.tensor(mine)
    gathered = [torch.empty_like(ids) for _ in range(world)]
    dist.all_gather(gathered, ids)
    t = torch.tensor([10.0 + rank])           # per-rank "elapsed ms"
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        allids = sorted(int(v) for g in gathered for v in g if v >= 0)
        q.put((allids, float(t)))
    dist.destroy_process_group()


def test_two_rank_stream_sharding():
    world, n = 2, 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    allids, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert allids == list(range(n))            # disjoint, complete cover
    assert tmax == 11.0                         # max over ranks


def test_route_preserves_stream_order():
    reqs = [(s % 5, i) for i, s in enumerate(range(40))]
    by_rank = route(reqs, 2)
    for r, items in by_rank.items():
        assert all(owner(sid, 2) == r for sid, _ in items)
        for sid in {s for s, _ in items}:
            seq = [i for s, i in items if s == sid]
            assert seq == sorted(seq)
