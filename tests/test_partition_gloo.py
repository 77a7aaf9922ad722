"""Multi-GPU shape of the path: independent decode streams,
partitioned across ranks with NO data-path collective. Exercised here on CPU
with world_size 2 over gloo: each rank builds its own stream (seed 7+rank),
runs the decision path (oracle) on it, and the only communication is the
bench's barrier + max/sum reductions of timings and counts."""
import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    sys.path.insert(0, REPO)
    import torch
    import pyoracle as po
    from paper_2508_18983_b200 import capi
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, E, B, T = 2, 64, 1, 24
    scores = capi.generate_trace(L, E, B, T, 7 + rank)  # the bench's per-rank stream
    out = po.simulate(po.SimCfg(num_layers=L, experts=E, top_k=6, batch=B, seed=7), scores, timeline=False)
    hits = torch.tensor([float(out["metrics"]["hits"]), float(out["metrics"]["selections"])])
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(hits, op=dist.ReduceOp.SUM)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    q.put((rank, out["metrics"]["hits"], out["metrics"]["selections"], hits.tolist(), t.item()))
    dist.destroy_process_group()


def test_two_rank_stream_partition():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, h0, s0, agg0, t0), (r1, h1, s1, agg1, t1) = res
    assert agg0 == agg1 == [float(h0 + h1), float(s0 + s1)]  # aggregate = sum of independent streams
    assert t0 == t1 == 2.0  # max over ranks
    # each rank's decisions equal a standalone run on its own sub-stream
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import pyoracle as po
    from paper_2508_18983_b200 import capi
    for rank, h in ((0, h0), (1, h1)):
        sc = capi.generate_trace(2, 64, 1, 24, 7 + rank)
        assert po.simulate(po.SimCfg(num_layers=2, experts=64, top_k=6, batch=1, seed=7), sc,
                           timeline=False)["metrics"]["hits"] == h
