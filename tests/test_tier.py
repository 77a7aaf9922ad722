"""The HBM expert tier's host logic (paper_2508_18983_b200/tier.py), CPU only:
ownership covers every (layer, expert) exactly once, shard offsets are dense,
and the source table assembled from gathered shard bases (gloo, world 2 —
the exchange PeerTier does with CUDA IPC handles) is identical on every rank
and points every expert into its owner's shard."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_18983_b200 import tier


@pytest.mark.parametrize("n,world", [(26 * 64, 8), (26 * 64, 3), (5, 2), (1, 1)])
def test_ownership_and_offsets(n, world):
    seen = {}
    for r in range(world):
        offs = tier.shard_offsets(n, world, r, 100)
        assert sorted(offs.values()) == [100 * i for i in range(len(offs))]
        for j in offs:
            assert tier.owner(j, world) == r
            seen[j] = r
    assert sorted(seen) == list(range(n))


def _worker(rank, world, port, n, eb, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    base = 1 << 40 | rank << 32  # a stand-in for this rank's shard address
    bases = [None] * world
    dist.all_gather_object(bases, base)
    table = tier.source_table(bases, n, world, eb)
    gathered = [None] * world
    dist.all_gather_object(gathered, table)
    out[rank] = (bases, gathered[0] == gathered[1], table)
    dist.destroy_process_group()


def test_source_table_gloo_world2():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    n, eb, world = 26 * 64, 17301504, 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, n, eb, out), nprocs=world, join=True)
    for r in range(world):
        bases, same, table = out[r]
        assert same
        for j, p in enumerate(table):
            o = tier.owner(j, world)
            assert p == bases[o] + tier.shard_offsets(n, world, o, eb)[j]
