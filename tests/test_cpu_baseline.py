"""The CPU baseline (oracle/cpu_moe.c, bench.py's cpu_baseline and --impl
reference legs) computes the same layer as the pinned restatement: its weight
generator is bit-exact with moe_layer_ref.synth_tensor (and so with
csrc/weights.cuh), and one layer agrees with layer_forward within 1e-5
relative L2. CPU only."""
import ctypes as C
import os

import numpy as np
import pytest

import moe_layer_ref as ml
from conftest import REPO


@pytest.fixture(scope="module")
def cm():
    lib = C.CDLL(os.path.join(REPO, "oracle", "libcpumoe.so"))
    lib.cpu_synth.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p, C.c_int]
    lib.cpu_moe_layer.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_int]
    lib.cpu_bytes_touched.restype = C.c_uint64
    return lib


@pytest.mark.parametrize("tensor,n,fan_in", [(ml.tid_expert(3, 5, 0), 4096 + 7, 2048),
                                             (ml.tid_shared(1, 2), 1 << 16, 2816),
                                             (ml.tid_router(25), 64 * 256, 256)])
def test_cpu_synth_bit_exact(cm, tensor, n, fan_in):
    out = np.empty(n, dtype=np.uint16)
    cm.cpu_synth(7, tensor, n, fan_in, out.ctypes.data, 4)
    assert np.array_equal(out, ml.synth_tensor(7, tensor, n, fan_in))


@pytest.mark.parametrize("shared_gate,nthreads", [(False, 1), (True, 3), (False, 8)])
def test_cpu_layer_matches_restatement(cm, shared_gate, nthreads):
    d, F, S, E, layer = 512, 128, 256, 16, 2
    model = ml.SynthModel(d, F, S, E, seed=7, shared_gate=shared_gate)
    rng = np.random.default_rng(1)
    x = ml.f32_to_bf16_bits(rng.standard_normal(d).astype(np.float32))
    sel = [1, 4, 9, 15]
    scores = ml.router_scores(model, layer, x[None])[0]
    bits = {e: model.expert_bits(layer, e) for e in sel}
    sh = np.concatenate([ml.synth_tensor(7, ml.tid_shared(layer, m), S * d, d if m < 2 else S) for m in range(3)])
    router = ml.synth_tensor(7, ml.tid_router(layer), E * d, d)
    sg = ml.synth_tensor(7, ml.tid_shared_gate(layer), d, d) if shared_gate else None
    ptrs = (C.c_void_p * len(sel))(*[bits[e].ctypes.data for e in sel])
    wts = np.array([scores[e] for e in sel], dtype=np.float32)
    logits = np.zeros(E, np.float32)
    y = np.zeros(d, np.float32)
    xn = np.zeros(d, np.uint16)
    cm.cpu_bytes_touched()
    cm.cpu_moe_layer(x.ctypes.data, d, F, S, E, router.ctypes.data, sh.ctypes.data,
                     sg.ctypes.data if sg is not None else None, ptrs, wts.ctypes.data, len(sel),
                     logits.ctypes.data, y.ctypes.data, xn.ctypes.data, nthreads)
    yref = ml.layer_forward(model, layer, x[None], [sel], scores[None])[0]
    assert np.linalg.norm(y - yref) / np.linalg.norm(yref) <= 1e-5
    np.testing.assert_allclose(ml.softmax32(logits), scores, rtol=1e-5, atol=1e-7)
    assert cm.cpu_bytes_touched() == E * d * 2 + 3 * S * d * 2 + len(sel) * 3 * F * d * 2


@pytest.mark.parametrize("shared_gate,renorm,nthreads", [(False, 0, 1), (True, 0, 4), (False, 1, 8)])
def test_cpu_prefill_layer_matches_restatement(cm, shared_gate, renorm, nthreads):
    """cpu_moe_prefill_layer (the prefill CPU baseline): plain top-k of the
    oracle's scores, then the layer, against layer_forward for all tokens."""
    d, F, S, E, k, layer, N = 256, 128, 256 if not renorm else 0, 16, 4, 1, 40
    model = ml.SynthModel(d, F, S, E, seed=7, shared_gate=shared_gate)
    rng = np.random.default_rng(2)
    x = ml.f32_to_bf16_bits(rng.standard_normal((N, d)).astype(np.float32))
    experts = [model.expert_bits(layer, e) for e in range(E)]
    ptrs = (C.c_void_p * E)(*[b.ctypes.data for b in experts])
    sh = np.concatenate([ml.synth_tensor(7, ml.tid_shared(layer, m), S * d, d if m < 2 else S) for m in range(3)]) \
        if S else np.zeros(1, np.uint16)
    router = ml.synth_tensor(7, ml.tid_router(layer), E * d, d)
    sg = ml.synth_tensor(7, ml.tid_shared_gate(layer), d, d) if shared_gate else None
    xn = np.zeros((N, d), np.uint16)
    cm.cpu_moe_prefill_layer.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                         C.c_float, C.c_void_p, C.c_void_p, C.c_int]
    yc = np.zeros((N, d), np.float32)
    cm.cpu_moe_prefill_layer(x.ctypes.data, N, d, F, S, E, k, router.ctypes.data, sh.ctypes.data,
                             sg.ctypes.data if sg is not None else None, ptrs, renorm, 1.0, xn.ctypes.data,
                             yc.ctypes.data, nthreads)
    scores = ml.router_scores(model, layer, x)
    sel = [list(np.lexsort((np.arange(E), -s.astype(np.float64)))[:k]) for s in scores]
    y = ml.layer_forward(model, layer, x, sel, scores, renormalize=bool(renorm))
    assert np.linalg.norm(yc - y) / np.linalg.norm(y) <= 1e-5
    assert np.array_equal(xn, ml.f32_to_bf16_bits(ml.bf16_bits_to_f32(x) + yc))
