"""The C-ABI boundary (include/moesched_b200.h) on CPU: the product library
loads without a GPU/driver, exports every declared entry point, reports
device calls as CUDA errors (no CPU fallback), and keeps the host-side parts
(trace synthesis) working."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "moesched_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(moeb_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("moeb_create", "moeb_destroy", "moeb_step", "moeb_route", "moeb_classify", "moeb_balance",
                 "moeb_cache_admit", "moeb_simulate", "moeb_set_logits_trace", "moeb_get_metrics",
                 "moeb_get_decisions_json", "moeb_last_error", "moeb_predict_scores", "moeb_build_queue"):
        assert must in names


def test_library_loads_and_exports_every_symbol():
    from paper_2508_18983_b200 import capi
    lib = capi.lib()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert missing == []


def test_no_torch_types_in_the_abi():
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)  # declarations only
    assert "torch" not in src and "at::" not in src
    assert "cudaStream_t" not in src and "#include <cuda" not in src  # streams are opaque void*


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2508_18983_b200 import capi
    with pytest.raises(capi.MoebError) as ei:
        capi.route(np.ones((1, 8)) / 8, np.zeros(8, dtype=np.uint8), 2, 0.1)
    assert ei.value.code == 5


def test_config_errors_are_reported_before_device_work():
    from paper_2508_18983_b200 import capi
    with pytest.raises(capi.MoebError) as ei:
        capi.simulate(capi.Config.make(num_layers=1, experts=8, top_k=8), np.zeros((1, 1, 1, 8)))
    assert ei.value.code == 1 and "k + 1 <= E required" in ei.value.msg
    with pytest.raises(capi.MoebError) as ei:
        capi.simulate(capi.Config.make(num_layers=1, experts=8, top_k=2, alpha=1.0), np.zeros((1, 1, 1, 8)))
    assert "router.alpha" in ei.value.msg
    with pytest.raises(capi.MoebError) as ei:
        capi.simulate(capi.Config.make(num_layers=1, experts=128, top_k=2, slots=4), np.zeros((1, 1, 1, 128)))
    assert "<= 64" in ei.value.msg


def test_host_trace_generator_invariants():  # test_trace.cpp:28-47, 55-65
    from paper_2508_18983_b200 import capi
    t = capi.generate_trace(2, 16, 2, 50, 3)
    assert t.shape == (50, 2, 2, 16)
    assert (t >= 0).all() and (t.sum(-1) <= 1 + 1e-6).all()
    assert capi.generate_trace(2, 8, 1, 0, 3).shape[0] == 0
    pin = capi.generate_trace(1, 16, 1, 40, 11, hot_fraction=1 / 16, persistence=1.0)
    tops = {int(np.argmax(pin[i, 0, 0])) for i in range(40)}
    assert len(tops) == 1
    assert np.array_equal(capi.generate_trace(2, 16, 1, 20, 7), capi.generate_trace(2, 16, 1, 20, 7))
    assert not np.array_equal(capi.generate_trace(2, 16, 1, 20, 7), capi.generate_trace(2, 16, 1, 20, 8))
