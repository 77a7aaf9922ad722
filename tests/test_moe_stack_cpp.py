"""The C++ real-layer API (include/moesched/moe_layer.hpp, moesched::MoeStack
in libmoesched.so) driven by a C++ caller on the B200
(tests/cpp/moe_stack_main.cpp, built by csrc/Makefile): the per-step
decisions it returns in the reference's RouteResult / load-list vocabulary,
replayed by the oracle on the router scores the device used, are bit-exact;
Metrics agree; pending is the reference's kept-low-and-not-resident set
(router.cpp:150, 250-258); a bad config raises ConfigError through the
wrapper, and MoeStack::prefill uploads exactly the non-resident experts and
returns bitwise-reproducible outputs without touching the decisions (the
program checks these itself)."""
import json
import os
import subprocess

import numpy as np
import pytest

import pyoracle as po
from conftest import REPO

pytestmark = pytest.mark.gpu
BIN = os.path.join(REPO, "paper_2508_18983_b200", "csrc", "build", "moe_stack_main")


@pytest.mark.parametrize("L,E,k,B,d,F,S,slots,T,er,ba", [
    (2, 16, 4, 1, 256, 128, 256, 4, 16, 1, 1),
    (2, 16, 4, 3, 256, 128, 256, 4, 12, 1, 1),
    (3, 64, 6, 8, 512, 128, 256, 16, 8, 1, 0),
])
def test_cpp_moe_stack_decisions_bit_exact(L, E, k, B, d, F, S, slots, T, er, ba):
    assert os.path.exists(BIN), "build with make -C paper_2508_18983_b200/csrc"
    r = subprocess.run([BIN] + [str(v) for v in (L, E, k, B, d, F, S, slots, T, er, ba)], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout)
    sc = np.array(out["scores"], dtype=np.float32).reshape(T, L, B, E).astype(np.float64)
    kw = dict(num_layers=L, experts=E, top_k=k, batch=B, slots=slots, alpha=0.25, seed=7, er=er, ba=ba)
    ref = po.simulate(po.SimCfg(**kw), sc, steps=True)
    got = out["steps"]
    for g in got:
        kept = sorted({e for t in g["tok"] for e in t["kept"]})
        assert g.pop("pending") == [e for e in kept if e not in g["mask"]]
    assert got == ref["steps"]
    for key in ("hits", "misses", "selections", "demand_loads", "cpu_computed", "prefetch_loads", "substitutions",
                "low_score_kept", "iterations", "total_time"):
        assert out["metrics"][key] == ref["metrics"][key], key
