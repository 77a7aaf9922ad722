"""CPU fp32 restatement of the MoE decode layer arithmetic — TEST INFRASTRUCTURE ONLY.

The reference abstracts expert compute as virtual tasks (pipeline.cpp:229-259,
SPEC.md:15), so this arithmetic has no reference implementation; it follows
the third-party model semantics the north star names (transformers 5.5.0):
  * DeepseekV2Moe (deepseek_v2/modeling_deepseek_v2.py:85-145): fp32 router
    logits, softmax, greedy top-k without renormalisation, x routed_scaling
    factor, plus shared experts;
  * Qwen2MoeSparseMoeBlock (qwen2_moe/modeling_qwen2_moe.py:334-370):
    sigmoid-gated shared expert;
  * MixtralSparseMoeBlock (mixtral/modeling_mixtral.py:101-119): top-k
    renormalised combine weights.
Expert choice is NOT recomputed here: the caller passes the device's
bit-exact decisions (checked separately against oracle/moesched_oracle.c),
and this module checks the arithmetic given those decisions.

Pinned: tests/test_hf_pin.py runs the installed HF modules (transformers 5.5.0)
on the same synthetic weights and activations and requires agreement within
1e-5 relative L2 (observed ~1.5e-7), plus RMSNorm within one bf16 ulp.

Weights are regenerated with the counter hash of
paper_2508_18983_b200/csrc/weights.cuh (integer arithmetic, bit-exact).
"""
from __future__ import annotations

import numpy as np

M1 = np.uint64(0xbf58476d1ce4e5b9)
M2 = np.uint64(0x94d049bb133111eb)
G1 = np.uint64(0x9E3779B97F4A7C15)
G2 = np.uint64(0xD1B54A32D192ED03)


def tid_router(layer):
    return (layer << 20) | (0xFFFF << 4)


def tid_shared(layer, m):
    return (layer << 20) | (0xFFFE << 4) | m


def tid_shared_gate(layer):
    return (layer << 20) | (0xFFFD << 4)


def tid_expert(layer, e, m):
    return (layer << 20) | (e << 4) | m


def _mix64(z):
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def f32_to_bf16_bits(f):
    b = np.ascontiguousarray(f, dtype=np.float32).view(np.uint32)
    b = b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))
    return (b >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b):
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


_CPUMOE = None


def _cpumoe():
    """oracle/libcpumoe.so's threaded generator (bit-exact with synth_tensor's
    numpy path: tests/test_cpu_baseline.py), or None when not built."""
    global _CPUMOE
    if _CPUMOE is None:
        import ctypes as C
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libcpumoe.so")
        try:
            lib = C.CDLL(path)
            lib.cpu_synth.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p, C.c_int]
            _CPUMOE = lib
        except OSError:
            _CPUMOE = False
    return _CPUMOE or None


def synth_tensor_fast(seed, tensor, n, fan_in):
    lib = _cpumoe()
    if lib is None:
        return synth_tensor(seed, tensor, n, fan_in)
    import os
    out = np.empty(n, dtype=np.uint16)
    lib.cpu_synth(seed, tensor, n, fan_in, out.ctypes.data, min(16, os.cpu_count() or 1))
    return out


def synth_tensor(seed, tensor, n, fan_in, offset=0):
    """bf16 bits of tensor elements [offset, offset + n) (weights.cuh synth_weight)."""
    scale = np.float32(np.sqrt(3.0 / float(fan_in)))
    with np.errstate(over="ignore"):
        i = np.arange(offset, offset + n, dtype=np.uint64)
        z = _mix64(np.uint64(seed) ^ (np.uint64(tensor) * G1) ^ (i * G2))
    u = (z >> np.uint64(40)).astype(np.uint32).astype(np.float32) * np.float32(2.0 ** -24)
    w = (np.float32(2.0) * u - np.float32(1.0)) * scale
    return f32_to_bf16_bits(w.astype(np.float32))


class SynthModel:
    """Regenerates any weight of a stack created with weight_seed."""

    def __init__(self, d, ffn, shared_ffn, E, seed, shared_gate=False):
        self.d, self.F, self.S, self.E, self.seed, self.shared_gate = d, ffn, shared_ffn, E, seed, shared_gate
        self._cache = {}

    def _get(self, key, make):
        if key not in self._cache:
            self._cache[key] = make()
        return self._cache[key]

    def router(self, layer):
        return self._get(("r", layer), lambda: bf16_bits_to_f32(
            synth_tensor(self.seed, tid_router(layer), self.E * self.d, self.d)).reshape(self.E, self.d))

    def shared(self, layer):
        d, S = self.d, self.S

        def mk():
            g = bf16_bits_to_f32(synth_tensor_fast(self.seed, tid_shared(layer, 0), S * d, d)).reshape(S, d)
            u = bf16_bits_to_f32(synth_tensor_fast(self.seed, tid_shared(layer, 1), S * d, d)).reshape(S, d)
            dn = bf16_bits_to_f32(synth_tensor_fast(self.seed, tid_shared(layer, 2), S * d, S)).reshape(d, S)
            return g, u, dn
        return self._get(("s", layer), mk)

    def shared_gate_row(self, layer):
        return self._get(("sg", layer), lambda: bf16_bits_to_f32(
            synth_tensor(self.seed, tid_shared_gate(layer), self.d, self.d)))

    def expert(self, layer, e):
        d, F = self.d, self.F

        def mk():
            g = bf16_bits_to_f32(synth_tensor_fast(self.seed, tid_expert(layer, e, 0), F * d, d)).reshape(F, d)
            u = bf16_bits_to_f32(synth_tensor_fast(self.seed, tid_expert(layer, e, 1), F * d, d)).reshape(F, d)
            dn = bf16_bits_to_f32(synth_tensor_fast(self.seed, tid_expert(layer, e, 2), F * d, F)).reshape(d, F)
            return g, u, dn
        return self._get(("e", layer, e), mk)

    def expert_bits(self, layer, e):
        """Host-pool layout of one expert: [gate F*d][up F*d][down d*F] bf16 bits."""
        d, F = self.d, self.F
        return np.concatenate([synth_tensor(self.seed, tid_expert(layer, e, m), F * d, d if m < 2 else F)
                               for m in range(3)])


def rmsnorm_bf16(x_bits):
    """RMSNorm (eps 1e-6, unit weight) of bf16 rows -> bf16 bits (fp32 math)."""
    x = bf16_bits_to_f32(x_bits).astype(np.float32)
    inv = (1.0 / np.sqrt((x.astype(np.float64) ** 2).mean(-1, keepdims=True) + 1e-6)).astype(np.float32)
    return f32_to_bf16_bits(x * inv)


def softmax32(logits):
    z = np.asarray(logits, dtype=np.float64)
    z = np.exp(z - z.max(-1, keepdims=True))
    return (z / z.sum(-1, keepdims=True)).astype(np.float32)


def swiglu(u, g, up, dn):
    """silu(g.u) * (up.u) -> down; u fp32 [d] or [n, d]; weights fp32 (from bf16)."""
    u64 = u.astype(np.float64)
    gv = u64 @ g.astype(np.float64).T
    uv = u64 @ up.astype(np.float64).T
    h = (gv / (1.0 + np.exp(-gv))) * uv
    return h @ dn.astype(np.float64).T


def layer_forward(model: SynthModel, layer, x_bits, sel, scores, renormalize=False, routed_scale=1.0):
    """One MoE layer for B tokens given the device's selections.

    x_bits: [B, d] bf16 bits; sel: per-token list of selected experts (after
    substitution); scores: [B, E] fp32 router scores the device used.
    Returns y [B, d] float64 (shared + weighted routed experts).
    """
    u = bf16_bits_to_f32(rmsnorm_bf16(x_bits))
    B = u.shape[0]
    y = np.zeros((B, model.d), dtype=np.float64)
    if model.S:
        g, up, dn = model.shared(layer)
        for t in range(B):
            ys = swiglu(u[t], g, up, dn)
            if model.shared_gate:
                z = float(model.shared_gate_row(layer).astype(np.float64) @ u[t].astype(np.float64))
                ys = ys / (1.0 + np.exp(-z))
            y[t] += ys
    # per expert, every token that selected it at once (same arithmetic)
    users = {}
    for t in range(B):
        denom = sum(float(scores[t][e]) for e in sel[t]) if renormalize else 1.0
        for e in sel[t]:
            users.setdefault(e, []).append((t, float(scores[t][e]) / denom * routed_scale))
    for e in sorted(users):
        toks = [t for t, _ in users[e]]
        g, up, dn = model.expert(layer, e)
        ye = swiglu(u[toks], g, up, dn)
        for i, (t, w) in enumerate(users[e]):
            y[t] += w * ye[i]
    return y


def router_scores(model: SynthModel, layer, x_bits):
    u = bf16_bits_to_f32(rmsnorm_bf16(x_bits)).astype(np.float64)
    return softmax32(u @ model.router(layer).astype(np.float64).T)
