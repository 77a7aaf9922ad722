"""Pins the fp32 layer restatement (oracle/moe_layer_ref.py) to the third-party
model code it claims to restate: transformers 5.5.0's DeepseekV2Moe,
Qwen2MoeSparseMoeBlock and MixtralSparseMoeBlock and their
RMSNorm. The HF modules are instantiated at small dimensions, loaded with the
same counter-based synthetic weights the device stack generates
(moe_layer_ref.SynthModel, bit-exact with csrc/weights.cuh), and run on the
same normalised activations; the restatement, given the experts HF itself
picked, must agree within 1e-5 relative L2. CPU only (no device code)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

import moe_layer_ref as ml  # noqa: E402  (oracle, checker only)

TOL = 1e-5


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))


def _load_experts(experts, model, layer):
    """HF 3-D expert params: gate_up_proj [E][2F][d] (gate rows, then up rows),
    down_proj [E][d][F]."""
    with torch.no_grad():
        for e in range(model.E):
            g, u, dn = model.expert(layer, e)
            experts.gate_up_proj[e].copy_(_t(np.concatenate([g, u], 0)))
            experts.down_proj[e].copy_(_t(dn))


def _load_mlp(mlp, model, layer):
    g, u, dn = model.shared(layer)
    with torch.no_grad():
        mlp.gate_proj.weight.copy_(_t(g))
        mlp.up_proj.weight.copy_(_t(u))
        mlp.down_proj.weight.copy_(_t(dn))


def _inputs(B, d, seed):
    rng = np.random.default_rng(seed)
    x_bits = ml.f32_to_bf16_bits(rng.standard_normal((B, d)).astype(np.float32))
    u = ml.bf16_bits_to_f32(ml.rmsnorm_bf16(x_bits))  # what the device's gate phase feeds the experts
    return x_bits, u


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("B", [1, 3])
def test_deepseek_v2_moe_matches_restatement(B):
    from transformers.models.deepseek_v2 import modeling_deepseek_v2 as m
    from transformers.models.deepseek_v2.configuration_deepseek_v2 import DeepseekV2Config

    d, F, E, k, layer = 256, 64, 16, 6, 3
    cfg = DeepseekV2Config(hidden_size=d, moe_intermediate_size=F, n_routed_experts=E, num_experts_per_tok=k,
                           n_shared_experts=2, routed_scaling_factor=1.0, topk_method="greedy", n_group=1,
                           topk_group=1, hidden_act="silu", intermediate_size=4 * d)
    moe = m.DeepseekV2Moe(cfg).float().eval()
    model = ml.SynthModel(d, F, 2 * F, E, seed=7)
    _load_experts(moe.experts, model, layer)
    _load_mlp(moe.shared_experts, model, layer)
    with torch.no_grad():
        moe.gate.weight.copy_(_t(model.router(layer)))
    _, u = _inputs(B, d, 11 + B)
    with torch.no_grad():
        y_hf = moe(_t(u).view(1, B, d)).view(B, d).numpy()
        logits = torch.nn.functional.linear(_t(u), moe.gate.weight)
        idx, _ = moe.route_tokens_to_experts(logits.view(1, B, E))
    sel = [sorted(int(e) for e in idx[t]) for t in range(B)]
    x_bits, _ = _inputs(B, d, 11 + B)
    scores = ml.router_scores(model, layer, x_bits)
    # the restatement's router agrees with HF's on the expert choice
    assert sel == [sorted(np.argsort(-scores[t], kind="stable")[:k].tolist()) for t in range(B)]
    y = ml.layer_forward(model, layer, x_bits, sel, scores)
    assert _rel(y, y_hf) <= TOL


@pytest.mark.parametrize("B", [1, 4])
def test_qwen2_moe_block_matches_restatement(B):
    from transformers.models.qwen2_moe import modeling_qwen2_moe as m
    from transformers.models.qwen2_moe.configuration_qwen2_moe import Qwen2MoeConfig

    d, F, S, E, k, layer = 256, 64, 256, 12, 4, 1
    cfg = Qwen2MoeConfig(hidden_size=d, moe_intermediate_size=F, shared_expert_intermediate_size=S, num_experts=E,
                         num_experts_per_tok=k, norm_topk_prob=False, hidden_act="silu")
    blk = m.Qwen2MoeSparseMoeBlock(cfg).float().eval()
    model = ml.SynthModel(d, F, S, E, seed=9, shared_gate=True)
    _load_experts(blk.experts, model, layer)
    g, up, dn = model.shared(layer)
    with torch.no_grad():
        blk.shared_expert.gate_proj.weight.copy_(_t(g))
        blk.shared_expert.up_proj.weight.copy_(_t(up))
        blk.shared_expert.down_proj.weight.copy_(_t(dn))
        blk.shared_expert_gate.weight.copy_(_t(model.shared_gate_row(layer)).view(1, d))
        blk.gate.weight.copy_(_t(model.router(layer)))
    x_bits, u = _inputs(B, d, 21 + B)
    with torch.no_grad():
        y_hf = blk(_t(u).view(1, B, d)).view(B, d).numpy()
        _, _, idx = blk.gate(_t(u))
    sel = [sorted(int(e) for e in idx[t]) for t in range(B)]
    scores = ml.router_scores(model, layer, x_bits)
    y = ml.layer_forward(model, layer, x_bits, sel, scores)
    assert _rel(y, y_hf) <= TOL


@pytest.mark.parametrize("B", [1, 2])
def test_mixtral_block_matches_restatement(B):
    from transformers.models.mixtral import modeling_mixtral as m
    from transformers.models.mixtral.configuration_mixtral import MixtralConfig

    d, F, E, k, layer = 256, 128, 8, 2, 5
    cfg = MixtralConfig(hidden_size=d, intermediate_size=F, num_local_experts=E, num_experts_per_tok=k,
                        hidden_act="silu", router_jitter_noise=0.0)
    blk = m.MixtralSparseMoeBlock(cfg).float().eval()
    model = ml.SynthModel(d, F, 0, E, seed=13)
    _load_experts(blk.experts, model, layer)
    with torch.no_grad():
        blk.gate.weight.copy_(_t(model.router(layer)))
    x_bits, u = _inputs(B, d, 31 + B)
    with torch.no_grad():
        y_hf = blk(_t(u).view(1, B, d)).view(B, d).numpy()
        _, _, idx = blk.gate(_t(u))
    sel = [sorted(int(e) for e in idx[t]) for t in range(B)]
    scores = ml.router_scores(model, layer, x_bits)
    y = ml.layer_forward(model, layer, x_bits, sel, scores, renormalize=True)
    assert _rel(y, y_hf) <= TOL


def test_rmsnorm_matches_hf():
    """The gate phase's RMSNorm (eps 1e-6, unit weight, bf16 in/out) against
    DeepseekV2RMSNorm on bf16 rows: equal to within one bf16 ulp (HF uses
    rsqrt in fp32, the restatement 1/sqrt in fp64 then fp32)."""
    from transformers.models.deepseek_v2.modeling_deepseek_v2 import DeepseekV2RMSNorm

    d = 2048
    x_bits, _ = _inputs(8, d, 5)
    norm = DeepseekV2RMSNorm(d, eps=1e-6).eval()
    xt = torch.from_numpy(ml.bf16_bits_to_f32(x_bits)).to(torch.bfloat16)
    with torch.no_grad():
        hf = norm(xt).float().numpy()
    ours = ml.bf16_bits_to_f32(ml.rmsnorm_bf16(x_bits))
    ulp = np.abs(hf.view(np.int32) - ours.view(np.int32)) >> 16
    assert ulp.max() <= 1
    assert (ulp == 0).mean() > 0.99
