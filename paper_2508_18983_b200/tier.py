"""The HBM expert tier: experts that miss the capped
cache are uploaded from GPU memory — a peer GPU's HBM over NVLink 5 — instead
of the pinned host pool over PCIe.

The full expert pool is sharded over the ranks of one node: the flattened
(layer, expert) index j belongs to rank j % world (`owner`), which keeps its
experts in one HBM allocation (`shard_offsets`), filled from the host pool.
Every rank exports its allocation with CUDA IPC, the handles are exchanged
over gloo (no NCCL), every rank maps the others' allocations, and the
per-(layer, expert) device pointers go to moeb_set_expert_sources: the copy
engine then pulls a missed expert from the owning GPU (cudaMemcpyDefault over
NVLink). Decisions are unchanged — only where upload bytes come from.

`LocalTier` keeps the whole pool in this GPU's own HBM: the same code path on
one GPU (the bound of a tier faster than PCIe; what a 1-GPU box can measure).
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def owner(j: int, world: int) -> int:
    """Rank holding the flattened (layer, expert) index j."""
    return j % world


def shard_offsets(n: int, world: int, rank: int, expert_bytes: int) -> dict[int, int]:
    """Byte offset of each expert of `rank`'s shard inside its allocation."""
    return {j: i * expert_bytes for i, j in enumerate(range(rank, n, world))}


def source_table(bases: list[int], n: int, world: int, expert_bytes: int) -> list[int]:
    """Per flattened (layer, expert): the device address of its weights, given
    every rank's (mapped) shard base address."""
    offs = [shard_offsets(n, world, r, expert_bytes) for r in range(world)]
    return [bases[owner(j, world)] + offs[owner(j, world)][j] for j in range(n)]


class _Cudart:
    def __init__(self):
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                self.lib = C.CDLL(name)
                break
            except OSError:
                continue
        else:
            raise RuntimeError("libcudart not found")

    def check(self, rc, what):
        if rc != 0:
            raise RuntimeError(f"{what} failed: CUDA error {rc}")

    def malloc(self, n: int) -> int:
        p = C.c_void_p()
        self.check(self.lib.cudaMalloc(C.byref(p), C.c_size_t(n)), "cudaMalloc")
        return p.value

    def free(self, ptr: int):
        self.lib.cudaFree(C.c_void_p(ptr))

    def h2d(self, dst: int, src: int, n: int):
        self.check(self.lib.cudaMemcpy(C.c_void_p(dst), C.c_void_p(src), C.c_size_t(n), 1), "cudaMemcpy")

    class IpcHandle(C.Structure):  # cudaIpcMemHandle_t, passed by value
        _fields_ = [("reserved", C.c_char * 64)]

    def ipc_handle(self, ptr: int) -> bytes:
        h = self.IpcHandle()
        self.check(self.lib.cudaIpcGetMemHandle(C.byref(h), C.c_void_p(ptr)), "cudaIpcGetMemHandle")
        return C.string_at(C.addressof(h), 64)  # all 64 bytes (c_char arrays stop at NUL)

    def ipc_open(self, handle: bytes) -> int:
        p = C.c_void_p()
        h = self.IpcHandle.from_buffer_copy(handle)
        self.lib.cudaIpcOpenMemHandle.argtypes = [C.POINTER(C.c_void_p), self.IpcHandle, C.c_uint]
        self.check(self.lib.cudaIpcOpenMemHandle(C.byref(p), h, 1), "cudaIpcOpenMemHandle")  # lazy peer access
        return p.value

    def ipc_close(self, ptr: int):
        self.lib.cudaIpcCloseMemHandle(C.c_void_p(ptr))


def _fill(torch, buf, pool_ptr: int, idx: list[int], expert_bytes: int):
    """Copy experts `idx` (flattened) of the pinned host pool into buf, in order."""
    if not idx:
        return
    src = np.frombuffer((C.c_uint8 * ((max(idx) + 1) * expert_bytes)).from_address(pool_ptr), dtype=np.uint8)
    for i, j in enumerate(idx):
        buf[i * expert_bytes:(i + 1) * expert_bytes].copy_(
            torch.from_numpy(src[j * expert_bytes:(j + 1) * expert_bytes]), non_blocking=False)


class LocalTier:
    """The whole expert pool in this GPU's HBM (one allocation)."""

    def __init__(self, torch, stack, n: int):
        pool_ptr, eb = stack.host_pool()
        self.buf = torch.empty(n * eb, dtype=torch.uint8, device="cuda")
        _fill(torch, self.buf, pool_ptr, list(range(n)), eb)
        torch.cuda.synchronize()
        self.table = [self.buf.data_ptr() + j * eb for j in range(n)]
        stack.set_expert_sources(self.table)


class PeerTier:
    """The pool sharded over the node's GPUs, mapped into every rank with CUDA IPC.
    Each shard is its own cudaMalloc allocation (an IPC handle names a whole
    allocation, so the shard must start at its base)."""

    def __init__(self, torch, dist, stack, n: int):
        world, rank = dist.get_world_size(), dist.get_rank()
        pool_ptr, eb = stack.host_pool()
        mine = list(range(rank, n, world))
        self.rt = _Cudart()
        self.base = self.rt.malloc(max(1, len(mine)) * eb)
        for i, j in enumerate(mine):
            self.rt.h2d(self.base + i * eb, pool_ptr + j * eb, eb)
        handles = [None] * world
        dist.all_gather_object(handles, self.rt.ipc_handle(self.base))
        self.mapped = {}
        bases = []
        for r, h in enumerate(handles):
            if r == rank:
                bases.append(self.base)
            else:
                self.mapped[r] = self.rt.ipc_open(h)
                bases.append(self.mapped[r])
        self.table = source_table(bases, n, world, eb)
        stack.set_expert_sources(self.table)
        dist.barrier()

    def close(self, stack, dist):
        stack.set_expert_sources(None)
        dist.barrier()  # every rank stopped reading before the shards go away
        for p in self.mapped.values():
            self.rt.ipc_close(p)
        self.mapped = {}
        dist.barrier()
        self.rt.free(self.base)
