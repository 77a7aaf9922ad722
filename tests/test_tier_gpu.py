"""The HBM expert tier (moeb_set_expert_sources, paper_2508_18983_b200/tier.py)
on the B200: uploads pulled from GPU memory instead of the pinned host pool.

  * LocalTier (the whole pool in this GPU's HBM): the same trace gives the
    same decisions and bitwise-identical layer outputs as the host-pool run,
    for the batch-1 (split-K) and the batched (tcgen05) stacks, and the
    prefill uploads the same bytes and returns the same hidden states;
  * PeerTier across two processes sharing the one GPU (CUDA IPC handles
    exchanged over gloo — the multi-GPU mapping path, here without NVLink):
    decisions and outputs again identical to the host-pool run.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(capi, torch, B, tier=None, peer=None, seed=7, T=12):
    L, E, k, d, F, S, slots = 2, 16, 4, 256, 128, 256, 4
    kw = dict(num_layers=L, experts=E, top_k=k, batch=B, slots=slots, alpha=0.25, seed=seed)
    st = capi.Stack(capi.Config.make(**kw), d, F, S, weight_seed=seed, log_steps=True)
    st.set_logits_trace(capi.trace_logits(capi.generate_trace(L, E, B, T, seed)), T)
    keep = None
    if tier == "local":
        from paper_2508_18983_b200.tier import LocalTier
        keep = LocalTier(torch, st, L * E)
    elif tier == "peer":
        from paper_2508_18983_b200.tier import PeerTier
        keep = PeerTier(torch, peer, st, L * E)
    g = torch.Generator().manual_seed(seed)
    xs = torch.randn(T, B, d, generator=g).to(torch.bfloat16).cuda()
    y = torch.empty(B, d, dtype=torch.bfloat16, device="cuda")
    for i in range(T):
        st.step(xs[i].data_ptr(), y.data_ptr(), B)
    st.sync()
    xp = (torch.randn(64, d, generator=g) * 2).to(torch.bfloat16).cuda()
    yp = torch.empty_like(xp)
    up = st.prefill(xp.data_ptr(), yp.data_ptr(), 64)
    st.sync()
    res = dict(dec=st.decisions(), yl=st.layer_outputs(), h2d=st.io_stats()["h2d_bytes"], up=up,
               yp=yp.cpu().view(torch.int16).numpy().copy(), y=y.cpu().view(torch.int16).numpy().copy())
    if tier == "peer":
        keep.close(st, peer)
    st.close()
    return res


def _same(a, b):
    assert a["dec"] == b["dec"]
    assert np.array_equal(a["yl"], b["yl"]) and np.array_equal(a["y"], b["y"])
    assert a["h2d"] == b["h2d"] and a["up"] == b["up"]
    assert np.array_equal(a["yp"], b["yp"])


@pytest.mark.parametrize("B", [1, 2])
def test_local_tier_matches_host_pool(gpu, B):
    import torch
    _same(_run(gpu, torch, B), _run(gpu, torch, B, tier="local"))


def _peer_worker(rank, world, port, B, out):
    import torch
    import torch.distributed as dist
    from paper_2508_18983_b200 import capi
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = _run(capi, torch, B)
        b = _run(capi, torch, B, tier="peer", peer=dist)
        _same(a, b)
        out[rank] = "ok"
    except Exception as e:  # reported by the parent
        out[rank] = repr(e)
    dist.destroy_process_group()


def test_peer_tier_two_processes_one_gpu(gpu):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.get_context("spawn").Manager().dict()
    mp.spawn(_peer_worker, args=(2, port, 1, out), nprocs=2, join=True)
    assert dict(out) == {0: "ok", 1: "ok"}
