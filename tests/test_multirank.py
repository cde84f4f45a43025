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


def test_bench_gpus_flag_spawns_ranks():
    """``bench.py --gpus 2`` outside torchrun re-launches itself with two
    ranks (torch.distributed.run, 127.0.0.1) and reports n_gpus = 2 from the
    max-over-ranks timing path (--dry-run: gloo, no GPU work)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--dry-run", "--steps", "3"], capture_output=True, text=True,
                         timeout=300, check=True).stdout
    line = json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["streams_total"] == 16 and line["scaling"] == "weak"


def test_reference_arm_uses_the_gpu_arm_inputs():
    """The CPU reference arm and the GPU arm build their inputs from the same
    deterministic Workload (planes, GE-dropped shards): same_config."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import numpy as np
    import bench
    a = bench.Workload("t", 64, 96, range(3), ("ge",))
    b = bench.Workload("t", 64, 96, range(3), ("ge",))
    for c, L in ((3, 1024), (1, 512)):
        for s in range(3):
            assert np.array_equal(a.planes(c, s), b.planes(c, s))
            ja, jb = a.job(c, L, s, s), b.job(c, L, s, s)
            assert ja[0] == jb[0] and ja[1] == jb[1] and np.array_equal(ja[2], jb[2])
            assert not ja[2].all()                     # every stream needs recovery
    ref = bench.CpuReference(a, threads=2)
    ref.frame()
    ref.frame()
