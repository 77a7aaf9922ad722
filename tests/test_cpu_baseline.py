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
