"""Stream partitioning across GPUs (BASELINE.json configs[4]).

The decode path shards only as independent request streams: per-layer expert
caches are private state (cache.hpp:67-77), and requests interact only inside
one batch (route pass 1's top-score set C and coalesce_for_batching,
router.cpp:105-112,154-260). So the C5 workload — n_requests independent
decode streams at batch B on G GPUs — is partitioned with no data-path
collective:

  * the requests form n_requests / B batch groups; group j is the batch-B
    workload trace generate_trace(L, E, B, T, seed0 + j) (trace.cpp:106-151);
  * GPU g takes the contiguous block of groups [g n/G, (g+1) n/G) and decodes
    them one after another on its own stack (own cache, copy stream, PCIe
    link), so its decisions equal a reference simulate() over the
    concatenation of its groups' traces with shape.batch_size = B;
  * the aggregate is tokens/s = sum over GPUs (whole-job time = the max over
    ranks).

Host-side pinned pools: one replica per NUMA node. The lowest rank whose GPU
sits on a (host, node) creates and first-touches that node's /dev/shm
segment (with its CPU affinity set to the node's cores, so the pages land in
that node's memory) and fills it through its stack; every other rank maps its
own node's replica only after a barrier that follows every fill.
"""
from __future__ import annotations

import os

import numpy as np


def groups_of(n_requests: int, batch: int) -> int:
    if batch < 1 or n_requests % batch:
        raise ValueError(f"C5: {n_requests} requests do not split into batches of {batch}")
    return n_requests // batch


def partition(n_requests: int, batch: int, world: int, rank: int) -> list[int]:
    """Batch groups decoded by `rank`: a contiguous block, every group exactly once."""
    n = groups_of(n_requests, batch)
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank out of range")
    if n < world:
        raise ValueError(f"C5: batch {batch} leaves {n} groups for {world} GPUs (need B <= n_requests / G)")
    return list(range(n * rank // world, n * (rank + 1) // world))


def group_seed(group: int, seed0: int = 7) -> int:
    return seed0 + group


def sub_stream(capi, L: int, E: int, batch: int, tokens: int, groups: list[int], seed0: int = 7) -> np.ndarray:
    """Router scores of a rank's sub-stream: its groups' traces concatenated
    along the iteration axis, [len(groups) * tokens][L][B][E] fp64."""
    return np.concatenate([capi.generate_trace(L, E, batch, tokens, group_seed(g, seed0)) for g in groups], axis=0)


# ------------------------------------------------------------ NUMA placement

def device_numa_node(device: int) -> int:
    """NUMA node of a CUDA device (sysfs of its PCI function; -1 if unknown)."""
    try:
        import torch
        p = torch.cuda.get_device_properties(device)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            return int(f.read().strip())
    except Exception:
        return -1


def node_cpus(node: int) -> set[int] | None:
    """Cores of a NUMA node (sysfs cpulist), intersected with this process's allowed set."""
    if node < 0:
        return None
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            spec = f.read().strip()
    except OSError:
        return None
    cpus = set()
    for part in spec.split(","):
        if not part:
            continue
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    cpus &= os.sched_getaffinity(0)
    return cpus or None


def pool_groups(keys: list) -> dict:
    """Ranks grouped by the (host, NUMA node) key of their GPU (an unknown node, -1, is one group)."""
    g: dict = {}
    for r, k in enumerate(keys):
        g.setdefault(k, []).append(r)
    return g


def pool_owner(keys: list, rank: int) -> int:
    """The rank that creates and fills the pool replica `rank` maps."""
    return min(pool_groups(keys)[keys[rank]])


def bind_to_device_node(device: int) -> int:
    """Bind this process to the cores of its GPU's NUMA node (so pinned pools
    it allocates are first-touched in the memory next to the GPU's PCIe root);
    returns the node (-1: unknown, no binding)."""
    node = device_numa_node(device)
    cpus = node_cpus(node)
    if cpus:
        os.sched_setaffinity(0, cpus)
    return node


class NodePools:
    """One pinned expert pool replica per (host, NUMA node), shared by the
    ranks whose GPUs sit on that node. Setup-time collectives only (gloo):
    the pool owners fill their replicas, a barrier, an all_gather of the pool
    layout flags, then every other rank maps its node's replica.

    Every rank binds itself to its GPU's NUMA node cores (the copy thread its
    stack starts inherits the binding), so the owner's first touch of the
    /dev/shm pages places them in that node's memory.
    """

    def __init__(self, dist, device: int, tag: str):
        import socket
        self.dist = dist
        self.world = dist.get_world_size() if dist is not None else 1
        self.rank = dist.get_rank() if dist is not None else 0
        self.node = bind_to_device_node(device)
        me = (socket.gethostname(), self.node)
        if dist is not None:
            everyone = [None] * self.world
            dist.all_gather_object(everyone, me)
        else:
            everyone = [me]
        self.members = pool_groups(everyone)[me]
        self.owner = pool_owner(everyone, self.rank)
        self.is_owner = self.rank == self.owner
        self.tag = tag

    def stack(self, capi, cfg, name: str, pool_bytes: int, **kw):
        """This rank's stack over its node's replica `name` (created and
        filled by the node's owner with the stack's own layout)."""
        if self.dist is None:
            return capi.Stack(cfg, **kw)
        path = f"/dev/shm/moeb_{self.tag}_{name}_n{self.node}"
        st = mm = None
        flags = None
        if self.is_owner:
            with open(path, "wb") as f:
                f.truncate(pool_bytes)
            mm = np.memmap(path, dtype=np.uint8, mode="r+", shape=(pool_bytes,))
            st = capi.Stack(cfg, weights_host=(mm.ctypes.data, mm), fill_pool=True, **kw)
            flags = st.pool_flags()
        self.dist.barrier()  # every owner has filled its replica
        allf = [None] * self.world
        self.dist.all_gather_object(allf, flags)
        if not self.is_owner:
            mm = np.memmap(path, dtype=np.uint8, mode="r+", shape=(pool_bytes,))
            st = capi.Stack(cfg, weights_host=(mm.ctypes.data, mm), pool_flags=allf[self.owner], **kw)
        self.dist.barrier()  # every member has mapped it
        if self.is_owner:
            os.unlink(path)  # the mappings stay valid
        return st
