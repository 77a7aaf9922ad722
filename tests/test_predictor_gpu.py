"""The partial-forward predictor on
the B200: stage Pre in weight-driven mode, the prediction for layer l from
layer l-1's shared expert + resident hits (MOEB_MODEL_PREDICTOR).

  * decisions: the device's per-step records and counters — including the
    PredictorStats (supplied heads and their kinds against the true scores,
    issued, cancelled) — equal the oracle's simulate() replayed on the
    device's router scores with the device's predictions supplied
    (prefetch.cpp:43-49 pass-through), bit-exact;
  * arithmetic: each prediction equals softmax(router_l(RMSNorm(bf16(x_{l-1}
    + shared + resident hits)))) recomputed by the CPU oracle (within 2e-4);
  * the predictor beats chance at naming a true top-score expert.
"""
import numpy as np
import pytest

import moe_layer_ref as ml
import pyoracle as po

pytestmark = pytest.mark.gpu


def _run(gpu, torch, L, E, k, B, d, F, S, slots, T, t_load, seed=7):
    kw = dict(num_layers=L, experts=E, top_k=k, batch=B, slots=slots, alpha=0.25, seed=seed, t_load=t_load,
              ce=1, er=1, pre=1, ba=1)
    st = gpu.Stack(gpu.Config.make(**kw), d, F, S, weight_seed=seed, log_steps=True, predictor=True)
    g = torch.Generator().manual_seed(seed)
    xs = (torch.randn(T, B, d, generator=g) * 3).to(torch.bfloat16).cuda()
    y = torch.empty(B, d, dtype=torch.bfloat16, device="cuda")
    for i in range(T):
        st.step(xs[i].data_ptr(), y.data_ptr(), B)
    st.sync()
    return st, kw, xs


@pytest.mark.parametrize("B,d,F,S,serial", [(1, 256, 128, 256, "0"), (4, 256, 128, 256, "0"),
                                             (1, 256, 128, 256, "1")])
def test_predictor_decisions_and_arithmetic(gpu, B, d, F, S, serial, monkeypatch):
    import torch
    monkeypatch.setenv("MOEB_SERIAL", serial)  # serial: entry B of a step is published by the next one
    L, E, k, slots, T = 3, 16, 4, 4, 16
    st, kw, xs = _run(gpu, torch, L, E, k, B, d, F, S, slots, T, t_load=2)
    sc = st.scores().reshape(T, L, B, E).astype(np.float64)
    pr = st.pred_scores().reshape(T, L, B, E)
    has = ~np.isnan(pr[..., 0])
    assert has.sum() == (T * L - 1) * B  # every step but the very first was a prefetch target
    dec = st.decisions()
    ref = po.simulate(po.SimCfg(**kw), sc, pred=np.nan_to_num(pr).astype(np.float64), has_pred=has.astype(np.uint8),
                      steps=True)
    assert "error" not in ref
    assert dec == ref["steps"]
    m = st.metrics()
    for key, v in list(ref["metrics"].items()) + list(ref["stats"].items()):
        assert m[key] == v, key
    assert m["prefetch_loads"] > 0 and m["trace_supplied"] == has.sum() and m["draws"] == 0
    # the predictions of the last token's layers 1..L-1 from the CPU oracle
    model = ml.SynthModel(d, F, S, E, kw["seed"])
    yl = st.layer_outputs()
    x = xs[-1].cpu().view(torch.int16).numpy().view(np.uint16)
    for l in range(L):
        step = dec[(T - 1) * L + l]
        if l > 0:
            want = np.stack([ml.router_scores(model, l, xp)[0] for xp in x_pred])
            np.testing.assert_allclose(pr[T - 1, l], want, rtol=0, atol=2e-4)
        # this layer's partial forward: shared expert + the hits (resident before routing)
        hits = [[e for e in t["sel"] if e in step["mask"]] for t in step["tok"]]
        y_loc = ml.layer_forward(model, l, x, hits, sc[T - 1, l].astype(np.float32))
        x_pred = [ml.f32_to_bf16_bits(ml.bf16_bits_to_f32(x[t]) + y_loc[t].astype(np.float32))[None] for t in range(B)]
        x = ml.f32_to_bf16_bits(ml.bf16_bits_to_f32(x) + yl[l].astype(np.float32))
    st.close()


def test_predictor_accuracy_at_dsv2_lite_shape(gpu):
    """DeepSeek-V2-Lite widths, 4 layers, weight-driven: the predicted head
    is a true top-score expert far more often than chance (k/E ~ 9%)."""
    import torch
    st, kw, xs = _run(gpu, torch, 4, 64, 6, 1, 2048, 1408, 2816, 16, 24, t_load=100)
    m = st.metrics()
    assert m["trace_supplied"] == 24 * 4 - 1
    assert m["head_top"] / m["trace_supplied"] > 0.3
    st.close()


def test_predictor_needs_weight_driven_routing(gpu):
    cfg = gpu.Config.make(num_layers=2, experts=16, top_k=4, batch=1, slots=4, pre=1)
    st = gpu.Stack(cfg, 256, 128, 256, weight_seed=1, log_steps=True, predictor=True)
    with pytest.raises(gpu.MoebError) as ei:
        st.set_logits_trace(gpu.trace_logits(gpu.generate_trace(2, 16, 1, 4, 7)), 4)
    assert ei.value.code == 1
    st.close()
