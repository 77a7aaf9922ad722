#!/usr/bin/env python3
"""Generate golden decision fixtures from the REFERENCE library itself.

Runs the unmodified reference (oracle/_ref/libmoesched_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile) on seeded inputs and stores its
outputs under tests/golden/. Only this script touches the reference; the
fixtures travel with the repository so the GPU box (which has no
/root/reference) can check the CUDA path against reference-produced answers.

    make -C oracle && python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle"))
import pyoracle as po  # noqa: E402

# (name, SimCfg kwargs, trace (L, E, B, iters, seed, hot_fraction), quantize, pred)
CASES = [
    ("c1_dsv2lite_1layer", dict(num_layers=1, experts=64, top_k=6, batch=1, slots=16, seed=7), (1, 64, 1, 128, 7, 0.125), False, False),
    ("acceptance_L4_B3", dict(num_layers=4, experts=64, top_k=6, batch=3, slots=16, seed=7), (4, 64, 3, 120, 7, 0.125), False, False),
    ("acceptance_baseline", dict(num_layers=4, experts=64, top_k=6, batch=3, slots=16, seed=7, ce=0, er=0, pre=0, ba=0), (4, 64, 3, 120, 7, 0.125), False, False),
    ("qwen_E60_k4_B8", dict(num_layers=3, experts=60, top_k=4, batch=8, slots=15, seed=11, alpha=0.35), (3, 60, 8, 40, 11, 0.125), False, False),
    ("mixtral_E8_k2_c2", dict(num_layers=4, experts=8, top_k=2, batch=1, slots=2, seed=3), (4, 8, 1, 80, 3, 0.25), False, False),
    ("prefetch_active", dict(num_layers=2, experts=16, top_k=4, batch=2, slots=4, seed=5, t_load=4, t_cpu_token=3, p_top=0.7), (2, 16, 2, 60, 5, 0.25), False, False),
    ("supplied_pred", dict(num_layers=3, experts=16, top_k=3, batch=2, slots=5, seed=9, t_load=3), (3, 16, 2, 40, 9, 0.25), False, True),
    ("lru_seeded_fill", dict(num_layers=2, experts=32, top_k=4, batch=4, slots=6, seed=21, policy=1, init_fill=1), (2, 32, 4, 50, 21, 0.125), False, False),
    ("empty_fill_ties", dict(num_layers=2, experts=12, top_k=3, batch=3, slots=3, seed=4, init_fill=2, alpha=0.5), (2, 12, 3, 50, 4, 0.25), True, False),
    ("zero_slots", dict(num_layers=2, experts=16, top_k=4, batch=2, slots=0, seed=8), (2, 16, 2, 30, 8, 0.25), False, False),
    ("deferral_small_cache", dict(num_layers=1, experts=8, top_k=3, batch=4, slots=2, seed=12, t_route=2), (1, 8, 4, 60, 12, 0.25), False, False),
    ("single_layer_wrap_prefetch", dict(num_layers=1, experts=8, top_k=2, batch=2, slots=3, seed=13, t_load=2, window=1), (1, 8, 2, 60, 13, 0.25), False, False),
]


def quantize(s):
    q = np.round(s * 8) / 8 / (1 + 1e-12)
    return q / np.maximum(q.sum(-1, keepdims=True), 1)


def main():
    if po.ref() is None:
        sys.exit("oracle/_ref/libmoesched_ref.so missing: run `make -C oracle` with /root/reference present")
    index = {}
    for name, kw, (L, E, B, iters, seed, hf), quant, pred in CASES:
        scores = po.generate_trace(L, E, B, iters, seed, hot_fraction=hf, use_ref=True)
        if quant:
            scores = quantize(scores)
        p = hp = None
        if pred:
            p = po.generate_trace(L, E, B, iters, seed + 100, hot_fraction=hf, use_ref=True)
            hp = (np.random.RandomState(seed).rand(iters, L, B) < 0.5).astype(np.uint8)
        cfg = po.SimCfg(**kw)
        out = po.ref_simulate(cfg, scores, p, hp, timeline=True)
        assert "error" not in out, out
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), scores=scores,
                            **({"pred": p, "has_pred": hp} if pred else {}))
        with open(os.path.join(HERE, f"{name}.json"), "w") as f:
            json.dump({"config": kw, "expected": out}, f, separators=(",", ":"))
        index[name] = {"metrics": out["metrics"], "timeline_violations": out["timeline_violations"]}
        print(name, out["metrics"]["hit_rate"], out["metrics"]["prefetch_loads"], out["timeline_violations"])

    # route / coalesce on random batches (the reference's route() itself)
    rng = np.random.RandomState(20240401)
    cases = []
    for i in range(300):
        E = int(rng.randint(3, 65))
        k = int(rng.randint(1, min(7, E)))
        B = int(rng.randint(1, 9))
        s = rng.rand(B, E)
        if rng.rand() < 0.4:
            s = np.floor(s * 6)
        s = s / max(s.sum(), 1e-9)
        m = (rng.rand(E) < 0.4).astype(np.uint8)
        a = float([0, 0.1, 0.25, 0.5, 0.9][rng.randint(5)])
        co = bool(rng.randint(2))
        cases.append({"scores": s.tolist(), "mask": m.tolist(), "k": k, "alpha": a, "coalesce": co,
                      "expected": po.ref_route(s, m, k, a, co)})
    with open(os.path.join(HERE, "route_cases.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))

    # generate_trace digests (trace.cpp:106-151)
    digests = {}
    for (L, E, B, iters, seed) in [(2, 16, 2, 50, 3), (26, 64, 1, 16, 7), (24, 60, 8, 4, 11), (32, 8, 1, 8, 5)]:
        t = po.generate_trace(L, E, B, iters, seed, use_ref=True)
        digests[f"{L}_{E}_{B}_{iters}_{seed}"] = hashlib.sha256(t.tobytes()).hexdigest()
    index["trace_sha256"] = digests
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
