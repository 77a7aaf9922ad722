"""BASELINE.json configs at their real model shapes, on the B200.

configs[0] C1  DeepSeek-V2-Lite, 1 layer, batch 1, 128 tokens, 16-expert cache
configs[2] C3  Qwen1.5-MoE-A2.7B shape (60 experts top-4 + sigmoid-gated shared
               expert), batch 1-8, importance-threshold (alpha) sweep
configs[3] C4  Mixtral-8x7B shape (8 experts top-2, d 4096, ffn 14336,
               renormalised), 2-experts-per-layer cache, stage ablation ladder
configs[4] C5  independent decode streams, one handle each (driven from
               concurrent host threads, as one per GPU)

Every case: the device's per-step decisions are bit-exact against the oracle
replayed on the device's fp32 router scores (and, where the reference library
was built into oracle/_ref, against the reference simulate() itself), and the
layer outputs agree with the CPU fp32 oracle within 1e-3 relative L2. Layer
counts are reduced where a case only needs the per-layer behaviour (the
pinned pool of a full Mixtral stack is 90 GB); the shapes of each layer are
the real ones.
"""
import threading

import numpy as np
import pytest

import moe_layer_ref as ml
import pyoracle as po
from test_stack_gpu import OUT_RTOL, check_decisions, check_outputs, run_stack

pytestmark = pytest.mark.gpu

SHAPES = {
    "dsv2_lite": dict(E=64, k=6, d=2048, F=1408, S=2816, shared_gate=0, renorm=0),
    "qwen15_moe": dict(E=60, k=4, d=2048, F=1408, S=5632, shared_gate=1, renorm=0),
    "mixtral_8x7b": dict(E=8, k=2, d=4096, F=14336, S=0, shared_gate=0, renorm=1),
}


def _reference_metrics_agree(kw, scores):
    """The reference simulate() (oracle/_ref) on the device's scores, when built."""
    if po.ref() is None:
        return
    want = po.ref_simulate(po.SimCfg(**kw), scores)
    got = po.simulate(po.SimCfg(**kw), scores)
    assert got["metrics"] == want["metrics"] and got["windows"] == want["windows"]


def _run(gpu, shape, L, B, slots, iters, **extra):
    import torch
    s = SHAPES[shape]
    st, kw, xs, y = run_stack(gpu, torch, L, s["E"], s["k"], B, s["d"], s["F"], s["S"], slots, iters,
                              shared_gate=s["shared_gate"], renorm=s["renorm"], **extra)
    dec, gsc, m = check_decisions(st, kw, iters)
    _reference_metrics_agree(kw, gsc)
    return st, kw, xs, dec, gsc, m


def test_c1_dsv2_lite_one_layer_128_tokens(gpu):
    st, kw, xs, dec, gsc, m = _run(gpu, "dsv2_lite", 1, 1, 16, 128)
    s = SHAPES["dsv2_lite"]
    err = check_outputs(st, kw, xs, dec, gsc, s["d"], s["F"], s["S"])
    assert err <= OUT_RTOL
    assert 0.5 < m["hits"] / m["selections"] < 1.0  # the cache is exercised both ways
    assert m["demand_loads"] + m["cpu_computed"] > 0
    st.close()


@pytest.mark.parametrize("B", [1, 2, 4, 8])
def test_c3_qwen_shape_batches(gpu, B):
    st, kw, xs, dec, gsc, m = _run(gpu, "qwen15_moe", 2, B, 15, 12)
    s = SHAPES["qwen15_moe"]
    check_outputs(st, kw, xs, dec, gsc, s["d"], s["F"], s["S"], shared_gate=1)
    st.close()


@pytest.mark.parametrize("alpha", [0.0, 0.15, 0.35, 0.6])
def test_c3_qwen_shape_alpha_sweep(gpu, alpha):
    """Importance threshold sweep (cli.cpp:215-218 grid points) through the full
    stack: decisions exact at every alpha, outputs within tolerance."""
    st, kw, xs, dec, gsc, m = _run(gpu, "qwen15_moe", 2, 4, 15, 10, alpha=alpha)
    s = SHAPES["qwen15_moe"]
    check_outputs(st, kw, xs, dec, gsc, s["d"], s["F"], s["S"], shared_gate=1)
    if alpha == 0.0:
        assert m["substitutions"] == 0
    st.close()


def test_c3_alpha_sweep_decisions_24_layers(gpu):
    """The whole 13-point sweep (alpha 0..0.6 step 0.05) over a 24-layer Qwen
    trace at batch 8: the device decision engine against the oracle (and the
    reference library itself when oracle/_ref was built)."""
    scores = po.generate_trace(24, 60, 8, 12, 7)
    for i in range(13):
        kw = dict(num_layers=24, experts=60, top_k=4, batch=8, slots=15, alpha=0.05 * i, seed=7)
        got = gpu.simulate(gpu.Config.make(**kw), scores)
        want = po.simulate(po.SimCfg(**kw), scores)
        for key in ("metrics", "windows", "evictions", "cache_final"):
            assert got[key] == want[key], (i, key)
        _reference_metrics_agree(kw, scores)


@pytest.mark.parametrize("stages", [(0, 0, 0, 0), (1, 0, 0, 0), (1, 1, 0, 0), (1, 1, 1, 0), (1, 1, 1, 1)])
def test_c4_mixtral_shape_ladder(gpu, stages):
    """2 layers of 8 x 352 MB experts (5.6 GB pinned pool), 2 cache slots per
    layer: every upload is a 352 MB PCIe transfer. Decisions exact for each
    rung of the ablation ladder (pipeline.cpp:387-403)."""
    st, kw, xs, dec, gsc, m = _run(gpu, "mixtral_8x7b", 2, 1, 2, 6, stages=stages)
    io = st.io_stats()
    eb = 3 * 14336 * 4096 * 2
    assert io["h2d_bytes"] == (m["demand_loads"] + m["cpu_computed"] + m["prefetch_loads"]) * eb
    s = SHAPES["mixtral_8x7b"]  # outputs of both layers at every rung
    check_outputs(st, kw, xs, dec, gsc, s["d"], s["F"], 0, 0, 1)
    st.close()


@pytest.mark.parametrize("B", [2, 4])
def test_c4_mixtral_shape_batched_tensor_core_ffn(gpu, B):
    """The Mixtral shape at batch 2 / 4: the tcgen05 FFN over UMMA-tiled
    experts at d = 4096, ffn = 14336 (112 intermediate tiles, 64 K-blocks) with
    renormalised combine weights; decisions exact, both layers' outputs."""
    st, kw, xs, dec, gsc, m = _run(gpu, "mixtral_8x7b", 2, B, 2, 5)
    s = SHAPES["mixtral_8x7b"]
    check_outputs(st, kw, xs, dec, gsc, s["d"], s["F"], 0, 0, 1)
    st.close()


def test_c5_independent_streams_concurrent_handles(gpu):
    """Stream partitioning: two decode streams (different trace seeds), each
    with its own handle, cache, copy thread and pinned pool, stepped from two
    host threads at once. Each stream's decisions equal its own oracle run."""
    import torch
    s = SHAPES["dsv2_lite"]
    L, B, T = 2, 4, 10
    handles = []
    for seed in (7, 8):
        kw = dict(num_layers=L, experts=s["E"], top_k=s["k"], batch=B, slots=16, alpha=0.25, seed=seed)
        st = gpu.Stack(gpu.Config.make(**kw), s["d"], s["F"], s["S"], weight_seed=seed, log_steps=True)
        st.set_logits_trace(gpu.trace_logits(gpu.generate_trace(L, s["E"], B, T, seed)), T)
        xs = torch.randn(T, B, s["d"], generator=torch.Generator().manual_seed(seed)).to(torch.bfloat16).cuda()
        handles.append((st, kw, xs))
    errors = []

    def drive(st, xs):
        try:
            y = torch.empty(B, s["d"], dtype=torch.bfloat16, device="cuda")
            for i in range(T):
                st.step(xs[i].data_ptr(), y.data_ptr(), B)
            st.sync()
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=drive, args=(st, xs)) for st, _, xs in handles]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for st, kw, xs in handles:
        dec, gsc, m = check_decisions(st, kw, T)
        check_outputs(st, kw, xs, dec, gsc, s["d"], s["F"], s["S"])
        st.close()


@pytest.mark.parametrize("B", [16, 32])
def test_c5_batched_capped_cache_full_width(gpu, B):
    """C5 at the real DeepSeek-V2-Lite widths (d 2048, ffn 1408, shared 2816)
    with the capped 16/64 cache: the batched tcgen05 FFN (gate_up K-split at
    B <= 16, none above) with PCIe uploads in flight. Decisions exact, every
    layer output within 1e-3 of the CPU oracle."""
    st, kw, xs, dec, gsc, m = _run(gpu, "dsv2_lite", 2, B, 16, 8)
    s = SHAPES["dsv2_lite"]
    check_outputs(st, kw, xs, dec, gsc, s["d"], s["F"], s["S"])
    assert m["demand_loads"] + m["cpu_computed"] > 0
    st.close()
