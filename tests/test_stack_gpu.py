"""The MoE decode stack on the B200 (moeb_create / moeb_step through the C-ABI).

Parity bar (north star):
  * routing / substitution / cache hit-miss / eviction / prefetch / BA
    decisions: bit-exact — the device's per-step records and counters equal
    the oracle's simulate() replayed on the fp32 router scores the device
    produced (the oracle itself is pinned to the reference library in
    test_golden.py);
  * layer outputs: relative L2 error <= 1e-3 against the CPU fp32 oracle
    (oracle/moe_layer_ref.py) given those decisions (bf16 weights, fp32
    accumulate on both sides; observed ~1e-7).
"""
import numpy as np
import pytest

import moe_layer_ref as ml
import pyoracle as po

pytestmark = pytest.mark.gpu
OUT_RTOL = 1e-3


def run_stack(capi, torch, L, E, k, B, d, F, S, slots, iters, stages=(1, 1, 1, 1), shared_gate=0, renorm=0,
              seed=7, alpha=0.25, t_load=100, trace=True, window=16, init_fill=0):
    kw = dict(num_layers=L, experts=E, top_k=k, batch=B, slots=slots, alpha=alpha, seed=seed, window=window,
              ce=stages[0], er=stages[1], pre=stages[2], ba=stages[3], t_load=t_load, init_fill=init_fill)
    st = capi.Stack(capi.Config.make(**kw), d, F, S, shared_gate, renorm, 1.0, weight_seed=seed, log_steps=True)
    if trace:
        st.set_logits_trace(capi.trace_logits(capi.generate_trace(L, E, B, iters, seed)), iters)
    g = torch.Generator().manual_seed(seed)
    xs = torch.randn(iters, B, d, generator=g).to(torch.bfloat16).cuda()
    y = torch.empty(B, d, dtype=torch.bfloat16, device="cuda")
    for i in range(iters):
        st.step(xs[i].data_ptr(), y.data_ptr(), B)
    st.sync()
    return st, kw, xs, y


def check_decisions(st, kw, iters):
    L, B, E = kw["num_layers"], kw["batch"], kw["experts"]
    dec = st.decisions()
    gsc = st.scores().reshape(iters, L, B, E).astype(np.float64)
    ref = po.simulate(po.SimCfg(**kw), gsc, steps=True)
    assert "error" not in ref
    assert dec == ref["steps"]
    m = st.metrics()
    for key, v in list(ref["metrics"].items()) + list(ref["stats"].items()):
        assert m[key] == v, key
    return dec, gsc, m


def check_outputs(st, kw, xs, dec, gsc, d, F, S, shared_gate=0, renorm=0):
    L, iters = kw["num_layers"], xs.shape[0]
    model = ml.SynthModel(d, F, S, kw["experts"], kw["seed"], shared_gate=bool(shared_gate))
    yl = st.layer_outputs()
    import torch
    x = xs[-1].cpu().view(torch.int16).numpy().view(np.uint16)
    worst = 0.0
    for l in range(L):
        sel = [t["sel"] for t in dec[(iters - 1) * L + l]["tok"]]
        yref = ml.layer_forward(model, l, x, sel, gsc[iters - 1, l].astype(np.float32), renormalize=bool(renorm))
        err = np.linalg.norm(yl[l] - yref) / max(np.linalg.norm(yref), 1e-30)
        worst = max(worst, err)
        x = ml.f32_to_bf16_bits(ml.bf16_bits_to_f32(x) + yl[l].astype(np.float32))  # the device's residual chain
    assert worst <= OUT_RTOL, worst
    return worst


CASES = {
    # name: (L, E, k, B, d, F, S, slots, iters, extra)
    "dsv2_like_b1": (2, 16, 4, 1, 256, 128, 256, 4, 40, {}),
    "dsv2_like_b3": (2, 16, 4, 3, 256, 128, 256, 4, 40, {}),
    "mixtral_like_renorm": (3, 16, 2, 2, 256, 64, 0, 2, 30, {"renorm": 1}),
    "qwen_like_shared_gate_b8": (2, 60, 4, 8, 512, 128, 512, 15, 30, {"shared_gate": 1}),
    "prefetch_active_L1": (1, 8, 2, 4, 256, 128, 0, 2, 30, {"renorm": 1, "t_load": 3}),
    "zero_slots": (2, 16, 4, 2, 256, 128, 256, 0, 20, {}),
    "baseline_stages": (2, 16, 4, 1, 256, 128, 256, 4, 30, {"stages": (0, 0, 0, 0)}),
    "lru_seeded_b32": (2, 64, 6, 32, 256, 64, 128, 24, 12, {"stages": (0, 1, 1, 1), "init_fill": 1}),
    "window_beyond_smem": (2, 64, 6, 2, 256, 64, 128, 16, 20, {"window": 40}),
    # batched tensor-core FFN (ffn_umma.cuh): ffn / shared_ffn multiples of 128
    "umma_b32": (2, 64, 6, 32, 256, 128, 256, 24, 12, {"stages": (0, 1, 1, 1), "init_fill": 1}),
    "umma_b17_d512": (2, 16, 4, 17, 512, 256, 128, 8, 12, {}),
    "umma_b2_renorm": (2, 16, 2, 2, 256, 128, 0, 4, 20, {"renorm": 1}),
    "umma_b32_ksplit_dsplit": (1, 16, 4, 32, 1024, 640, 256, 8, 8, {}),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_stack_decisions_and_outputs(gpu, name):
    import torch
    L, E, k, B, d, F, S, slots, iters, extra = CASES[name]
    st, kw, xs, y = run_stack(gpu, torch, L, E, k, B, d, F, S, slots, iters, **extra)
    dec, gsc, m = check_decisions(st, kw, iters)
    check_outputs(st, kw, xs, dec, gsc, d, F, S, extra.get("shared_gate", 0), extra.get("renorm", 0))
    assert np.isfinite(y.float().cpu().numpy()).all()
    st.close()


def test_trace_mode_scores_reproduce_reference_trace(gpu):
    """softmax(ln s) on the device reproduces the reference trace scores."""
    import torch
    st, kw, xs, _ = run_stack(gpu, torch, 2, 64, 6, 1, 256, 64, 128, 16, 16)
    gsc = st.scores().reshape(16, 2, 1, 64).astype(np.float64)
    ref = gpu.generate_trace(2, 64, 1, 16, 7)
    np.testing.assert_allclose(gsc, ref / ref.sum(-1, keepdims=True), rtol=2e-6, atol=1e-12)
    st.close()


def test_weight_driven_router(gpu):
    """Without a logits trace the router GEMV drives routing; scores match the
    CPU oracle's fp32 router within tolerance and decisions stay bit-exact."""
    import torch
    L, E, B, d, F, S = 2, 16, 2, 256, 64, 128
    st, kw, xs, _ = run_stack(gpu, torch, L, E, 4, B, d, F, S, 4, 12, stages=(1, 1, 0, 1), trace=False)
    dec, gsc, _ = check_decisions(st, kw, 12)
    check_outputs(st, kw, xs, dec, gsc, d, F, S)
    model = ml.SynthModel(d, F, S, E, kw["seed"])
    yl = st.layer_outputs()
    x = xs[-1].cpu().view(torch.int16).numpy().view(np.uint16)
    for l in range(L):
        np.testing.assert_allclose(gsc[-1, l], ml.router_scores(model, l, x), rtol=1e-4, atol=1e-6)
        x = ml.f32_to_bf16_bits(ml.bf16_bits_to_f32(x) + yl[l].astype(np.float32))
    st.close()


def test_batch1_reset_replays(gpu):
    """Batch 1 (split-K FFN, rows dealt round-robin to the CTAs): decisions
    and layer outputs replay bit-for-bit after reset (with or without the
    MOEB_MODEL_DETERMINISTIC flag, which is the default behaviour)."""
    import torch
    L, E, k, d, F, S, T = 2, 16, 4, 256, 128, 256, 16
    xs = torch.randn(T, 1, d, generator=torch.Generator().manual_seed(3)).to(torch.bfloat16).cuda()
    for det in (False, True):
        kw = dict(num_layers=L, experts=E, top_k=k, batch=1, slots=4, alpha=0.25, seed=7)
        st = gpu.Stack(gpu.Config.make(**kw), d, F, S, weight_seed=7, log_steps=True, deterministic=det)
        st.set_logits_trace(gpu.trace_logits(gpu.generate_trace(L, E, 1, T, 7)), T)
        outs = []
        for rep in range(2):
            if rep:
                st.reset()
            y = torch.empty(T, 1, d, dtype=torch.bfloat16, device="cuda")
            for i in range(T):
                st.step(xs[i].data_ptr(), y[i].data_ptr(), 1)
            st.sync()
            outs.append((y.clone(), st.layer_outputs().copy()))
        dec = st.decisions()
        assert dec[:T * L] == dec[T * L:]
        assert torch.equal(outs[0][0], outs[1][0])
        assert np.array_equal(outs[0][1], outs[1][1])
        st.close()


def test_reset_replays_identically(gpu):
    import torch
    st, kw, xs, y = run_stack(gpu, torch, 2, 16, 4, 2, 256, 128, 256, 4, 20)
    d1, y1, m1 = st.decisions(), y.clone(), st.metrics()
    st.reset()
    y2 = torch.empty_like(y)
    for i in range(20):
        st.step(xs[i].data_ptr(), y2.data_ptr(), 2)
    st.sync()
    assert st.decisions()[len(d1):] == d1
    assert torch.equal(y1, y2)
    assert st.metrics() == m1
    st.close()


def test_api_errors(gpu):
    import torch
    cfg = gpu.Config.make(num_layers=1, experts=16, top_k=4, batch=2, slots=4, pre=1)
    st = gpu.Stack(cfg, 256, 64, 0, weight_seed=1)
    x = torch.zeros(2, 256, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(gpu.MoebError) as ei:
        st.step(x.data_ptr(), x.data_ptr(), 1)
    assert ei.value.code == 1 and "batch" in ei.value.msg
    with pytest.raises(gpu.MoebError) as ei:
        st.step(x.data_ptr(), x.data_ptr(), 2)
    assert "Pre needs a logits trace" in ei.value.msg
    st.close()
    with pytest.raises(gpu.MoebError):
        gpu.Stack(gpu.Config.make(num_layers=1, experts=16, top_k=4, batch=1), 100, 64, 0)


def _check_all_layers(st, dec, gsc, xs_step, step, model, L):
    import torch
    x = xs_step.cpu().view(torch.int16).numpy().view(np.uint16)
    yl = st.layer_outputs()
    worst = 0.0
    for l in range(L):
        sel = [t["sel"] for t in dec[step * L + l]["tok"]]
        yref = ml.layer_forward(model, l, x, sel, gsc[step, l].astype(np.float32))
        worst = max(worst, np.linalg.norm(yl[l] - yref) / np.linalg.norm(yref))
        x = ml.f32_to_bf16_bits(ml.bf16_bits_to_f32(x) + yl[l].astype(np.float32))
    assert worst <= OUT_RTOL, worst
    return worst


def test_dsv2_lite_full_stack(gpu):
    """The bench workload at full size (26 layers, d=2048, 64x17.3 MB experts
    per layer in a 28.8 GB pinned pool, cache 16/64): decisions bit-exact over
    24 tokens, uploads accounted, and every one of the 26 layer outputs of the
    last two tokens against the CPU oracle."""
    import torch
    L, T = 26, 24
    kw = dict(num_layers=L, experts=64, top_k=6, batch=1, slots=16, alpha=0.25, seed=7)
    st = gpu.Stack(gpu.Config.make(**kw), 2048, 1408, 2816, weight_seed=7, log_steps=True)
    st.set_logits_trace(gpu.trace_logits(gpu.generate_trace(L, 64, 1, T, 7)), T)
    xs = torch.randn(T, 1, 2048, generator=torch.Generator().manual_seed(7)).to(torch.bfloat16).cuda()
    y = torch.empty(1, 2048, dtype=torch.bfloat16, device="cuda")
    model = ml.SynthModel(2048, 1408, 2816, 64, 7)
    for i in range(T):
        st.step(xs[i].data_ptr(), y.data_ptr(), 1)
        if i >= T - 2:
            st.sync()
            dec = st.decisions()
            gsc = st.scores().reshape(i + 1, L, 1, 64).astype(np.float64)
            _check_all_layers(st, dec, gsc, xs[i], i, model, L)
    st.sync()
    dec, gsc, m = check_decisions(st, kw, T)
    io = st.io_stats()
    eb = 3 * 1408 * 2048 * 2
    # every decided upload moved once: by its own copy, or (promoted) by the
    # speculative upload that anticipated it; wasted speculation on top
    assert io["h2d_bytes"] - io["spec_bytes"] + io["spec_promoted"] * eb == \
        (m["demand_loads"] + m["cpu_computed"] + m["prefetch_loads"]) * eb
    assert m["demand_loads"] + m["cpu_computed"] > 0  # the capped cache really uploads
    st.close()


@pytest.mark.parametrize("B", [1, 4])
def test_serial_mode_matches_pipelined(gpu, B, monkeypatch):
    """Serial (profiler-safe) mode — MOEB_SERIAL=1, automatic under ncu /
    nsys / compute-sanitizer: upload dependencies as host-set stream waits,
    no in-kernel spins on a concurrent engine. Same decisions, same outputs
    (to fp32 reassociation: item order may differ) as the pipelined mode."""
    import torch
    runs = []
    for serial in ("0", "1"):
        monkeypatch.setenv("MOEB_SERIAL", serial)
        st, kw, xs, y = run_stack(gpu, torch, 2, 16, 4, B, 256, 128, 256, 4, 20)
        dec, gsc, m = check_decisions(st, kw, 20)
        check_outputs(st, kw, xs, dec, gsc, 256, 128, 256)
        runs.append((dec, y.float().cpu().numpy(), m))
        st.close()
    assert runs[0][0] == runs[1][0] and runs[0][2] == runs[1][2]
    np.testing.assert_allclose(runs[1][1], runs[0][1], rtol=2e-2, atol=2e-2)  # bf16 hidden of the last step


def test_decision_log_overflow_is_loud(gpu):
    """The per-step log keeps the first 16384 layer-steps; past that,
    decisions()/scores() fail instead of returning a truncated log."""
    import torch
    L, T = 64, 260  # 16640 layer-steps
    kw = dict(num_layers=L, experts=8, top_k=2, batch=1, slots=8, alpha=0.25, seed=7)
    st = gpu.Stack(gpu.Config.make(**kw), 256, 64, 0, weight_seed=7, log_steps=True)
    st.set_logits_trace(gpu.trace_logits(gpu.generate_trace(L, 8, 1, T, 7)), T)
    x = torch.randn(1, 256).to(torch.bfloat16).cuda()
    y = torch.empty_like(x)
    for i in range(T):
        st.step(x.data_ptr(), y.data_ptr(), 1)
    st.sync()
    with pytest.raises(gpu.MoebError) as ei:
        st.decisions()
    assert ei.value.code == 4 and "overflow" in ei.value.msg
    with pytest.raises(gpu.MoebError):
        st.scores()
    st.close()


def test_speculative_uploads_keep_decisions_and_outputs(gpu, monkeypatch):
    """MOEB_SPEC_UPLOAD=1 (opt-in): the next layer's likely miss is uploaded
    into a side buffer while the copy engine idles and used when that upload
    is decided. Decisions and outputs are those of the default path; every
    decided upload moved exactly once (by its own copy or the buffer)."""
    import torch
    monkeypatch.setenv("MOEB_SPEC_UPLOAD", "1")
    L, E, k, d, F, S, slots, T = 3, 16, 4, 256, 128, 256, 4, 40
    st, kw, xs, y = run_stack(gpu, torch, L, E, k, 1, d, F, S, slots, T)
    dec, gsc, m = check_decisions(st, kw, T)
    check_outputs(st, kw, xs, dec, gsc, d, F, S)
    io = st.io_stats()
    eb = 3 * F * d * 2
    assert io["spec_jobs"] > 0 and io["spec_promoted"] > 0
    assert io["h2d_bytes"] - io["spec_bytes"] + io["spec_promoted"] * eb == \
        (m["demand_loads"] + m["cpu_computed"] + m["prefetch_loads"]) * eb
    st.close()
