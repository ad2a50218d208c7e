"""Multi-rank host logic of bench.py on CPU (gloo, world size 2): disjoint per-rank workloads
(weak scaling, no data-path collective) and the max-over-ranks timing reduction."""
import os
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    lo, hi = bench.rank_seed_range(rank, 4096)
    t = bench.max_over_ranks(10.0 + rank)  # rank 1 is slower
    out.put((rank, lo, hi, t))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, lo0, hi0, t0), (r1, lo1, hi1, t1) = res
    assert (lo0, hi0) == (0, 4096) and (lo1, hi1) == (4096, 8192)  # disjoint seeds
    assert t0 == t1 == 11.0                                         # max over ranks on every rank
