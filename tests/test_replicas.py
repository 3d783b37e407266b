"""Multi-GPU replica logic of bench.py on CPU with gloo, world_size 2.

The path does not shard within one source ("replicas only"): each rank solves its own
source on its own copy of the graph, and the only collectives are the barrier and the
max-over-ranks reduction of the timings.  These tests cover that host logic without a GPU.
"""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import gen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, out):
    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    g = gen.make("rmat12")
    src = bench.replica_source(g, rank)
    t = bench.max_over_ranks(10.0 * (rank + 1), ws, dist)
    dist.barrier()
    out[rank] = (src, t)
    dist.destroy_process_group()


def test_replicas_gloo_world2():
    ws = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, _free_port(), out), nprocs=ws, join=True)
    g = gen.make("rmat12")
    (s0, t0), (s1, t1) = out[0], out[1]
    assert s0 == g.source  # rank 0 runs the workload's source
    assert 0 <= s1 < g.n and g.degrees[s1] > 0 and s1 != s0
    assert t0 == t1 == 20.0  # the slowest rank decides, on every rank


def test_replica_sources_deterministic():
    import bench

    g = gen.make("grid64")
    assert [bench.replica_source(g, r) for r in range(4)] == [bench.replica_source(g, r) for r in range(4)]
    assert bench.max_over_ranks(3.5, 1) == 3.5
