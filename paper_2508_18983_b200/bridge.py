"""Wire-format bridge between a B200 decode run and the reference's tools
(SURVEY.md section 8(f) rank 2).

* export_trace(): the router scores the device actually computed (widened to
  fp64, as the decision engine uses them) written as the reference's GateTrace
  JSONL (trace.cpp:153-181: a {"L","E","k","B"} header, then one
  {"it","layer","tok","s"} record per (iteration, layer, token)), so the
  reference's own load_trace()/simulate() can replay a B200 run.
* report(): the run's metrics and predictor statistics in the reference's
  single-run report schema (report.cpp:19-83: metrics_to_json,
  prefetch_stats_to_json, trace_fingerprint = FNV-1a of the trace file,
  trace.cpp:353-372).

Host-side only: both read what the stack already logged (MOEB_MODEL_LOG_STEPS).
"""
from __future__ import annotations

import json

import numpy as np


def fingerprint_bytes(data: bytes) -> str:
    """FNV-1a 64 (trace.cpp:353-362)."""
    h = 0xcbf29ce484222325
    for c in data:
        h ^= c
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def _fnv_file(path: str) -> str:
    with open(path, "rb") as f:
        return fingerprint_bytes(f.read())


def export_trace(stack, cfg: dict, path: str, iterations: int | None = None) -> int:
    """Write the device's fp32 router scores as a reference GateTrace JSONL.

    cfg: the Config.make(**cfg) keywords of the stack (num_layers, experts,
    top_k, batch). Returns the number of iterations written.
    """
    L, E, k, B = cfg["num_layers"], cfg["experts"], cfg["top_k"], cfg["batch"]
    sc = stack.scores().astype(np.float64)
    T = sc.size // (L * B * E)
    if iterations is not None:
        T = min(T, iterations)
    sc = sc[:T * L * B * E].reshape(T, L, B, E)
    with open(path, "w") as f:
        f.write(json.dumps({"L": L, "E": E, "k": k, "B": B}, separators=(",", ":")) + "\n")
        for it in range(T):
            for layer in range(L):
                for t in range(B):
                    rec = {"it": it, "layer": layer, "tok": t, "s": [float(v) for v in sc[it, layer, t]]}
                    f.write(json.dumps(rec, separators=(",", ":")) + "\n")
    return T


def stage_label(cfg: dict) -> str:
    """StageSet::label (core.cpp:11-24)."""
    names = [n for key, n in (("ce", "CE"), ("er", "ER"), ("pre", "Pre"), ("ba", "BA")) if cfg.get(key, 1)]
    return "+".join(names) if names else "baseline"


def report(stack, cfg: dict, trace_path: str | None = None) -> dict:
    """The run in the reference's report schema (metrics + prefetch_stats +
    trace fingerprint). Values are the device's own counters."""
    m = stack.metrics()
    metrics = {"stage": stage_label(cfg)}
    for key in ("tpot", "hit_rate", "substitution_ratio", "demand_loads", "prefetch_loads", "cpu_computed", "hits",
                "misses", "substitutions", "low_score_kept", "selections", "iterations", "total_time"):
        metrics[key] = m[key]
    total = m["draws"] + m["trace_supplied"]
    non_top = m["head_active"] + m["head_inactive"]
    stats = {"draws": m["draws"], "trace_supplied": m["trace_supplied"], "head_top": m["head_top"],
             "head_active": m["head_active"], "head_inactive": m["head_inactive"],
             "head_accuracy": 0.0 if total == 0 else m["head_top"] / total,
             "active_rate": 0.0 if non_top == 0 else m["head_active"] / non_top,
             "issued": m["issued"], "cancelled": m["cancelled"]}
    out = {"metrics": metrics, "prefetch_stats": stats}
    if trace_path:
        out["trace_fingerprint"] = _fnv_file(trace_path)
    return out
