"""Multi-GPU shape of the path: independent decode streams,
partitioned across ranks with NO data-path collective. Runs the product's own
partitioning and pool-placement code (paper_2508_18983_b200/partition.py, as
bench.py uses it) on CPU with world_size 2 over gloo:

  * partition(): the C5 workload (64 requests at batch B) splits into
    contiguous blocks of batch groups, every group exactly once;
  * sub_stream(): each rank's router-score stream is its groups' traces
    back to back, and the decisions on it (oracle = checker) equal a
    reference simulate() of that sub-stream (per-GPU decisions are a
    standalone run, nothing crosses ranks);
  * NodePools: one pinned-pool replica per (host, NUMA node): its owner
    creates and fills it, the other rank maps it only after the barrier that
    follows the fill, with the owner's layout flags; the segment is unlinked.
The stacks are stand-ins here (no GPU); the GPU side of the same path is the
bench's c5_partitioned section and test_configs_gpu.py's concurrent handles.
"""
import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class _FakeStack:
    """Records how NodePools creates a stack (no device)."""

    def __init__(self, cfg, weights_host=None, fill_pool=False, pool_flags=0, **kw):
        self.ptr, self.mm = weights_host
        self.fill, self.flags_in = fill_pool, pool_flags
        if fill_pool:
            self.mm[:16] = np.arange(16, dtype=np.uint8)  # "weights"
        self.seen = bytes(self.mm[:16])

    def pool_flags(self):
        return 8  # MOEB_MODEL_DOWN_T


class _FakeCapi:
    Stack = _FakeStack


def _worker(rank, world, port, q):
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    sys.path.insert(0, REPO)
    import torch
    import pyoracle as po
    from paper_2508_18983_b200 import capi, partition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, E, B, T = 2, 64, 8, 5
    groups = partition.partition(64, B, world, rank)
    scores = partition.sub_stream(capi, L, E, B, T, groups)
    out = po.simulate(po.SimCfg(num_layers=L, experts=E, top_k=6, batch=B, seed=7), scores, timeline=False)
    allg = [None] * world
    dist.all_gather_object(allg, groups)
    hits = torch.tensor([float(out["metrics"]["hits"]), float(out["metrics"]["selections"])])
    dist.all_reduce(hits, op=dist.ReduceOp.SUM)
    # pool placement
    pools = partition.NodePools(dist, 0, f"test{port}")
    st = pools.stack(_FakeCapi, None, "rows", 4096)
    path = f"/dev/shm/moeb_test{port}_rows_n{pools.node}"
    dist.barrier()
    q.put((rank, groups, allg, out["metrics"]["hits"], out["metrics"]["selections"], hits.tolist(),
           pools.is_owner, st.fill, st.flags_in, st.seen, os.path.exists(path)))
    dist.destroy_process_group()


def test_two_rank_stream_partition_and_node_pool():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1 = res
    # contiguous blocks covering all 8 groups exactly once, agreed by both ranks
    assert r0[2] == r1[2] == [r0[1], r1[1]]
    assert sorted(r0[1] + r1[1]) == list(range(8)) and r0[1] == [0, 1, 2, 3]
    # aggregate = sum of the independent streams
    assert r0[5] == r1[5] == [float(r0[3] + r1[3]), float(r0[4] + r1[4])]
    # each rank's decisions: a standalone reference-equivalent run of its sub-stream
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import pyoracle as po
    from paper_2508_18983_b200 import capi
    for r in res:
        groups, hits, sel = r[1], r[3], r[4]
        sc = np.concatenate([capi.generate_trace(2, 64, 8, 5, 7 + g) for g in groups])
        cfg = po.SimCfg(num_layers=2, experts=64, top_k=6, batch=8, seed=7)
        want = (po.ref_simulate if po.ref() is not None else po.simulate)(cfg, sc)
        assert want["metrics"]["hits"] == hits and want["metrics"]["selections"] == sel
    # node pool: one owner filled, the other mapped the filled replica with its flags; unlinked after
    owners = [r for r in res if r[6]]
    assert len(owners) == 1 and owners[0][0] == 0
    assert r0[7] is True and r1[7] is False and r1[8] == 8
    assert r0[9] == r1[9] == bytes(range(16))
    assert not r0[10] and not r1[10]


def test_partition_rejects_oversized_batches():
    sys.path.insert(0, REPO)
    from paper_2508_18983_b200 import partition
    assert partition.partition(64, 32, 2, 1) == [1]
    with pytest.raises(ValueError):
        partition.partition(64, 32, 4, 0)  # B <= 64 / G
    with pytest.raises(ValueError):
        partition.partition(64, 3, 1, 0)
    keys = [("a", 0), ("a", 1), ("a", 0), ("b", 0)]
    assert [partition.pool_owner(keys, r) for r in range(4)] == [0, 1, 0, 3]
