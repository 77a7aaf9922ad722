"""Prefill (moeb_prefill) on the B200:
N prompt tokens per layer, plain top-k routing, the grouped tcgen05 GEMM
behind a warp-aggregated token -> expert permutation (prefill.cuh).

Per layer, from the prefill log:
  * router scores = softmax(router(RMSNorm(x))) recomputed by the CPU oracle
    (within 2e-4);
  * selections = the reference's plain_top_k (router.cpp:252-260: score
    descending, index ascending) of the device's scores, bit-exact;
  * the fp32 layer output = oracle/moe_layer_ref.layer_forward (pinned to the
    HF modules, tests/test_hf_pin.py) given those selections, within 1e-3
    relative L2;
  * the residual chain: layer l+1's input = bf16(x_l + y_l) bit-exact, and
    the returned hidden is the last layer's.
Also: bitwise-reproducible outputs, the decode state untouched, uploads of
exactly the non-resident experts, batch-1 (row-interleaved) stacks through
the re-tiling pass, and the shape requirement.
"""
import numpy as np
import pytest

import moe_layer_ref as ml
from test_stack_gpu import OUT_RTOL

pytestmark = pytest.mark.gpu


def _plain_top_k(sc, k):
    E = sc.shape[-1]
    return np.stack([np.lexsort((np.arange(E), -row.astype(np.float64)))[:k] for row in sc])


def _run(gpu, torch, L, E, k, B, d, F, S, slots, N, shared_gate=0, renorm=0, seed=7, routed_scale=1.0):
    cfg = gpu.Config.make(num_layers=L, experts=E, top_k=k, batch=B, slots=slots, seed=seed)
    st = gpu.Stack(cfg, d, F, S, shared_gate, renorm, routed_scale, weight_seed=seed, log_steps=True)
    g = torch.Generator().manual_seed(seed + N)
    x = (torch.randn(N, d, generator=g) * 2).to(torch.bfloat16).cuda()
    y = torch.empty(N, d, dtype=torch.bfloat16, device="cuda")
    up = st.prefill(x.data_ptr(), y.data_ptr(), N)
    st.sync()
    return st, x, y, up


def _check(st, x, y, L, E, k, d, F, S, shared_gate, renorm, seed, routed_scale=1.0, tokens=None):
    import torch
    model = ml.SynthModel(d, F, S, E, seed, shared_gate=bool(shared_gate))
    xin0 = x.cpu().view(torch.int16).numpy().view(np.uint16)
    worst = 0.0
    prev = None
    for l in range(L):
        xi, sc, sel, yl = st.prefill_log(l)
        if l == 0:
            assert np.array_equal(xi, xin0)
        else:  # the residual chain, bit-exact
            assert np.array_equal(xi, ml.f32_to_bf16_bits(ml.bf16_bits_to_f32(prev[0]) + prev[1]))
        assert np.array_equal(sel, _plain_top_k(sc, k))
        idx = np.arange(xi.shape[0]) if tokens is None else tokens
        want_sc = ml.router_scores(model, l, xi[idx])
        np.testing.assert_allclose(sc[idx], want_sc, rtol=0, atol=2e-4)
        yref = ml.layer_forward(model, l, xi[idx], [list(map(int, s)) for s in sel[idx]], sc[idx],
                                renormalize=bool(renorm), routed_scale=routed_scale)
        err = np.linalg.norm(yl[idx] - yref) / max(np.linalg.norm(yref), 1e-30)
        worst = max(worst, err)
        prev = (xi, yl)
    out = y.cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(out, ml.f32_to_bf16_bits(ml.bf16_bits_to_f32(prev[0]) + prev[1]))
    assert worst <= OUT_RTOL, worst
    return worst


CASES = {
    # name: (L, E, k, B, d, F, S, slots, N, shared_gate, renorm)
    "dsv2_like_one_token": (2, 16, 4, 2, 256, 128, 256, 4, 1, 0, 0),
    "dsv2_like_37": (2, 16, 4, 2, 256, 128, 256, 4, 37, 0, 0),
    "dsv2_like_300_multi_tile": (2, 16, 4, 2, 256, 128, 256, 4, 300, 0, 0),
    "qwen_like_shared_gate": (2, 60, 4, 2, 512, 128, 512, 15, 96, 1, 0),
    "mixtral_like_renorm_no_shared": (2, 8, 2, 2, 256, 256, 0, 2, 200, 0, 1),
    "all_resident": (2, 16, 4, 2, 256, 128, 256, 16, 64, 0, 0),
    "zero_slots": (1, 16, 4, 2, 256, 128, 256, 0, 50, 0, 0),
    # batch-1 stacks keep experts row-interleaved (split-K decode): prefill re-tiles them
    "dsv2_like_b1_rows": (2, 16, 4, 1, 256, 128, 256, 4, 77, 0, 0),
    "qwen_like_b1_rows": (2, 60, 4, 1, 512, 128, 512, 15, 40, 1, 0),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_prefill_matches_oracle(gpu, name):
    import torch
    L, E, k, B, d, F, S, slots, N, sg, rn = CASES[name]
    st, x, y, up = _run(gpu, torch, L, E, k, B, d, F, S, slots, N, sg, rn)
    _check(st, x, y, L, E, k, d, F, S, sg, rn, 7)
    # uploads: exactly the experts outside the cache, every layer
    assert up == L * (E - min(slots, E)) * 3 * F * d * 2
    st.close()


def test_prefill_reproducible_and_decode_state_untouched(gpu):
    import torch
    L, E, k, B, d, F, S, slots, N = 2, 16, 4, 2, 256, 128, 256, 4, 150
    st, x, y, _ = _run(gpu, torch, L, E, k, B, d, F, S, slots, N)
    m0 = st.metrics()
    y2 = torch.empty_like(y)
    st.prefill(x.data_ptr(), y2.data_ptr(), N)
    st.sync()
    assert torch.equal(y.view(torch.int16), y2.view(torch.int16))
    assert st.metrics() == m0
    st.close()


def test_prefill_right_after_decode_with_prefetches(gpu):
    """Decode steps whose stage Pre issues prefetches (copies into cache slots
    that land after the step), then a prefill at once: it must read every
    resident slot only after its upload landed, and match the oracle."""
    import torch
    L, E, k, B, d, F, S, slots, T, N = 1, 8, 2, 4, 256, 128, 0, 2, 30, 50
    kw = dict(num_layers=L, experts=E, top_k=k, batch=B, slots=slots, alpha=0.25, seed=7, t_load=3)
    st = gpu.Stack(gpu.Config.make(**kw), d, F, S, 0, 1, 1.0, weight_seed=7, log_steps=True)
    st.set_logits_trace(gpu.trace_logits(gpu.generate_trace(L, E, B, T, 7)), T)
    g = torch.Generator().manual_seed(3)
    xs = torch.randn(T, B, d, generator=g).to(torch.bfloat16).cuda()
    yd = torch.empty(B, d, dtype=torch.bfloat16, device="cuda")
    for i in range(T):
        st.step(xs[i].data_ptr(), yd.data_ptr(), B)
    x = (torch.randn(N, d, generator=g) * 2).to(torch.bfloat16).cuda()
    y = torch.empty_like(x)
    st.prefill(x.data_ptr(), y.data_ptr(), N)  # no sync in between
    st.sync()
    assert st.metrics()["prefetch_loads"] > 0
    _check(st, x, y, L, E, k, d, F, S, 0, 1, 7)
    st.close()


@pytest.mark.parametrize("B", [1, 2])
def test_prefill_dsv2_lite_full_width(gpu, B):
    """DeepSeek-V2-Lite widths (64 experts top-6, 2 shared, d 2048, ffn 1408),
    2 layers, a 512-token prompt, cache 16/64, on a batch-1 (re-tiled) and a
    batched stack: every layer's scores and selections for all tokens,
    outputs of 48 tokens against the oracle."""
    import torch
    L, E, k, d, F, S, slots, N = 2, 64, 6, 2048, 1408, 2816, 16, 512
    st, x, y, up = _run(gpu, torch, L, E, k, B, d, F, S, slots, N)
    assert up == L * 48 * 3 * F * d * 2
    rng = np.random.default_rng(0)
    _check(st, x, y, L, E, k, d, F, S, 0, 0, 7, tokens=np.sort(rng.choice(N, 48, replace=False)))
    st.close()


@pytest.mark.parametrize("shape", ["qwen15_moe", "mixtral_8x7b"])
def test_prefill_full_width_shapes(gpu, shape):
    """Qwen1.5-MoE (60 experts top-4, 5632-wide sigmoid-gated shared expert)
    and Mixtral-8x7B (d 4096, ffn 14336, renormalised top-2, no shared expert)
    at full width, one layer on a batched stack with the capped cache: scores,
    selections and the residual chain for every token, outputs of 16 tokens
    against the oracle."""
    import torch
    L, E, k, d, F, S, sg, rn, slots, N = {
        "qwen15_moe": (1, 60, 4, 2048, 1408, 5632, 1, 0, 15, 128),
        "mixtral_8x7b": (1, 8, 2, 4096, 14336, 0, 0, 1, 2, 48)}[shape]
    st, x, y, up = _run(gpu, torch, L, E, k, 2, d, F, S, slots, N, sg, rn)
    assert up == L * (E - slots) * 3 * F * d * 2
    rng = np.random.default_rng(1)
    _check(st, x, y, L, E, k, d, F, S, sg, rn, 7, tokens=np.sort(rng.choice(N, 16, replace=False)))
    st.close()


def test_prefill_needs_128_multiple_ffn(gpu):
    import torch
    cfg = gpu.Config.make(num_layers=1, experts=16, top_k=4, batch=1, slots=4)
    st = gpu.Stack(cfg, 256, 64, 256, weight_seed=1)  # ffn 64: no tensor-core tiling
    x = torch.zeros(4, 256, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(gpu.MoebError) as ei:
        st.prefill(x.data_ptr(), x.data_ptr(), 4)
    assert ei.value.code == 1
    st.close()
