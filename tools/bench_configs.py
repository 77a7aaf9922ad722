#!/usr/bin/env python3
"""Every named shape of BASELINE.json at 1 GPU, through the same code path as
bench.py (moeb_create / moeb_step through the C-ABI, trace-driven routing,
PCIe uploads from the pinned pool on the copy stream):

  C1  DeepSeek-V2-Lite, 1 layer, batch 1, 128 tokens, 16-expert cache; the
      5-stage ablation ladder (pipeline.cpp:387-403)
  C2  the headline (bench.py) — not repeated here
  C3  Qwen1.5-MoE-A2.7B shape (24 layers, 60 experts top-4, sigmoid-gated
      shared expert 5632), cache 15/60, batch 1/2/4/8, and the 13-point alpha
      sweep 0..0.6 (cli.cpp:215-218) at batch 4
  C4  Mixtral-8x7B shape (32 layers, 8 experts top-2, d 4096, ffn 14336,
      renormalised), 2-expert cache per layer, batch 1, the ablation ladder
  C5  64 independent DeepSeek-V2-Lite requests stream-partitioned
      (partition.py) at batch 1..32 on this one GPU, cache 16/64

Per case: ms per decode step and tokens/s (CUDA events on the stack's
stream, after warm-up), hit rate, uploads, the path roofline
T_roof = max(B_hbm / BW_hbm, B_pcie / BW_pcie) with BW_pcie measured here, and
(for the headline rung of C1/C3/C4) the CPU path on this host's cores
(bench.cpu_path). Prints one JSON object; --out writes it to a file.

  python tools/bench_configs.py --out gpurun_out/configs.json [--only C1,C4]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402  (helpers: ar1_hidden, peaks, measure_pcie_gbs, cpu_path, c5_partitioned)

DSV2 = dict(experts=64, top_k=6, d_model=2048, ffn=1408, shared_ffn=2816, shared_gate=0, renormalize=0)
QWEN = dict(experts=60, top_k=4, d_model=2048, ffn=1408, shared_ffn=5632, shared_gate=1, renormalize=0)
MIXTRAL = dict(experts=8, top_k=2, d_model=4096, ffn=14336, shared_ffn=0, shared_gate=0, renormalize=1)
LADDER = [("baseline", (0, 0, 0, 0)), ("CE", (1, 0, 0, 0)), ("CE+ER", (1, 1, 0, 0)), ("CE+ER+Pre", (1, 1, 1, 0)),
          ("CE+ER+Pre+BA", (1, 1, 1, 1))]


def split(shape):
    cfg = dict(experts=shape["experts"], top_k=shape["top_k"])
    model = {k: shape[k] for k in ("d_model", "ffn", "shared_ffn", "shared_gate", "renormalize")}
    model["routed_scale"] = 1.0
    return cfg, model


def run_case(capi, torch, cfg_d, model_d, T, K, hbm_peak, pcie_peak, pool=None, seed=7, setup=None):
    """Decode a T-token stream, time its last K steps. Returns (row, stack).
    setup(stack), if given, runs before the first step."""
    L, E, B, d = cfg_d["num_layers"], cfg_d["experts"], cfg_d["batch"], model_d["d_model"]
    scores = capi.generate_trace(L, E, B, T, seed)
    x = torch.from_numpy(bench.ar1_hidden(T, B, d, seed)).to(torch.bfloat16).cuda()
    y = torch.empty((B, d), dtype=torch.bfloat16, device="cuda")
    cfg = capi.Config.make(**cfg_d)
    kw = {}
    if pool is not None:
        kw["weights_host"] = (pool.host_pool()[0], pool)
    t0 = time.time()
    st = capi.Stack(cfg, weight_seed=7, **kw, **model_d)
    create_s = time.time() - t0
    st.set_logits_trace(capi.trace_logits(scores), T)
    keep = setup(st) if setup else None
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(T - K):
            st.step(x[i].data_ptr(), y.data_ptr(), B, stream=s.cuda_stream)
        st.sync()
        m0, io0 = st.metrics(), st.io_stats()
        st.reset_kernel_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(T - K, T):
            st.step(x[i].data_ptr(), y.data_ptr(), B, stream=s.cuda_stream)
        st.sync()  # every upload the timed steps published has landed (they are counted)
        e1.record(s)
        e1.synchronize()
    ms = e0.elapsed_time(e1) / K
    m1, io1, ks = st.metrics(), st.io_stats(), st.kernel_stats()
    sel = m1["selections"] - m0["selections"]
    b_hbm = (ks["ffn_bytes"] + ks["route_bytes"]) / K
    eb = 3 * model_d["ffn"] * d * 2
    b_pcie = (io1["h2d_bytes"] - io1["spec_bytes"] + io1["spec_promoted"] * eb) / K  # io counters zeroed above
    t_roof = max(b_hbm / (hbm_peak * 1e9), b_pcie / (pcie_peak * 1e9)) * 1e3
    row = {"ms_per_step": round(ms, 4), "tokens_per_s": round(B * 1e3 / ms, 1),
           "ms_per_token": round(ms / B, 4), "hit_rate": round((m1["hits"] - m0["hits"]) / max(sel, 1), 4),
           "demand_loads": m1["demand_loads"] - m0["demand_loads"],
           "streamed_ba": m1["cpu_computed"] - m0["cpu_computed"],
           "prefetch_loads": m1["prefetch_loads"] - m0["prefetch_loads"],
           "substitutions": m1["substitutions"] - m0["substitutions"],
           "path_roofline": {"t_roof_ms": round(t_roof, 4), "frac": round(t_roof / ms, 4),
                             "hbm_mb_per_step": round(b_hbm / 1e6, 1), "pcie_mb_per_step": round(b_pcie / 1e6, 1),
                             "bound": "pcie" if b_pcie / pcie_peak > b_hbm / hbm_peak else "hbm",
                             "pcie_busy_frac": round(io1["copy_ms"] / (ms * K), 4)},
           "steps_timed": K, "stream_steps": T, "create_s": round(create_s, 1)}
    return row, st, scores


def cpu_row(cfg_d, model_d, scores, T, n_tokens):
    B, d = cfg_d["batch"], model_d["d_model"]
    x_host = bench.ar1_hidden(T, B, d, 7)
    ms, kind, cores, sample, gbs = bench.cpu_path(scores, x_host, n_tokens, os.cpu_count() or 1, cfg_d, model_d)
    return {"value": round(ms, 3), "unit": "ms/step", "cores": cores, "kind": kind, "sample": sample,
            "host_weight_gbs": round(gbs, 1)}


def c1(capi, torch, hbm, pcie, cpu):
    cfg, model = split(DSV2)
    out = {"workload": "DeepSeek-V2-Lite, 1 layer, batch 1, 128 tokens, cache 16/64, alpha 0.25", "ladder": {}}
    pool = None
    for name, (ce, er, pre, ba) in LADDER:
        cfg_d = dict(cfg, num_layers=1, batch=1, slots=16, alpha=0.25, seed=7, ce=ce, er=er, pre=pre, ba=ba)
        row, st, scores = run_case(capi, torch, cfg_d, model, 128, 96, hbm, pcie, pool)
        if name == "CE+ER+Pre+BA" and cpu:
            row["cpu_baseline"] = cpu_row(cfg_d, model, scores, 128, 96)
        out["ladder"][name] = row
        if pool is None:
            pool = st
        else:
            st.close()
    pool.close()
    return out


def c3(capi, torch, hbm, pcie, cpu):
    cfg, model = split(QWEN)
    out = {"workload": "Qwen1.5-MoE-A2.7B shape, 24 layers, cache 15/60, CE+ER+Pre+BA", "batch": {}, "alpha_sweep_B4": {}}
    pools = {}
    for B in (1, 2, 4, 8):
        cfg_d = dict(cfg, num_layers=24, batch=B, slots=15, alpha=0.25, seed=7)
        key = "b1" if B == 1 else "tiled"
        row, st, scores = run_case(capi, torch, cfg_d, model, 64, 48, hbm, pcie, pools.get(key))
        if B == 1 and cpu:
            row["cpu_baseline"] = cpu_row(cfg_d, model, scores, 64, 4)
        out["batch"][f"B{B}"] = row
        if key not in pools:
            pools[key] = st
        else:
            st.close()
    for i in range(13):
        alpha = round(0.05 * i, 2)
        cfg_d = dict(cfg, num_layers=24, batch=4, slots=15, alpha=alpha, seed=7)
        row, st, _ = run_case(capi, torch, cfg_d, model, 48, 32, hbm, pcie, pools["tiled"])
        out["alpha_sweep_B4"][str(alpha)] = {k: row[k] for k in ("ms_per_step", "tokens_per_s", "hit_rate",
                                                                 "substitutions", "demand_loads", "streamed_ba")}
        st.close()
    for p in pools.values():
        p.close()
    return out


def c4(capi, torch, hbm, pcie, cpu):
    cfg, model = split(MIXTRAL)
    out = {"workload": "Mixtral-8x7B shape, 32 layers, batch 1, cache 2/8 per layer (90 GB pinned pool)", "ladder": {}}
    pool = None
    for name, (ce, er, pre, ba) in LADDER:
        cfg_d = dict(cfg, num_layers=32, batch=1, slots=2, alpha=0.25, seed=7, ce=ce, er=er, pre=pre, ba=ba)
        row, st, scores = run_case(capi, torch, cfg_d, model, 12, 8, hbm, pcie, pool)
        if name == "CE+ER+Pre+BA" and cpu:
            row["cpu_baseline"] = cpu_row(cfg_d, model, scores, 12, 1)
        out["ladder"][name] = row
        if pool is None:
            pool = st
        else:
            st.close()
    pool.close()
    return out


def c2_predictor(capi, torch, hbm, pcie, cpu):
    """The headline shape in weight-driven mode: routing from the router GEMV
    on the hidden stream, stage Pre fed by the paper's partial-forward
    predictor (MOEB_MODEL_PREDICTOR). Reports ms/token and the prefetch
    accuracy in the reference's PredictorStats vocabulary (prefetch.hpp:68-88):
    the predicted head's class against the true scores of that step."""
    cfg, model = split(DSV2)
    L, E, B, d, T, K = 26, 64, 1, 2048, 64, 48
    out = {"workload": "DeepSeek-V2-Lite 26 L, batch 1, cache 16/64, weight-driven routing, stage Pre with the "
                       "partial-forward predictor (shared expert + resident hits -> next layer's router)"}
    res = {}
    for name, pred in (("predictor", True), ("pre_off", False)):
        cfg_d = dict(cfg, num_layers=L, batch=B, slots=16, alpha=0.25, seed=7, pre=1 if pred else 0)
        st = capi.Stack(capi.Config.make(**cfg_d), weight_seed=7, predictor=pred, **model)
        x = torch.from_numpy(bench.ar1_hidden(T, B, d, 7)).to(torch.bfloat16).cuda()
        y = torch.empty((B, d), dtype=torch.bfloat16, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for i in range(T - K):
                st.step(x[i].data_ptr(), y.data_ptr(), B, stream=s.cuda_stream)
            st.sync()
            m0 = st.metrics()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for i in range(T - K, T):
                st.step(x[i].data_ptr(), y.data_ptr(), B, stream=s.cuda_stream)
            st.sync()  # every upload the timed steps published has landed (they are counted)
            e1.record(s)
            e1.synchronize()
        m1 = st.metrics()
        dm = {k: m1[k] - m0[k] for k in m1 if isinstance(m1[k], int)}
        sel = max(dm["selections"], 1)
        row = {"ms_per_token": round(e0.elapsed_time(e1) / K, 4), "hit_rate": round(dm["hits"] / sel, 4),
               "demand_loads": dm["demand_loads"], "streamed_ba": dm["cpu_computed"],
               "prefetch_loads": dm["prefetch_loads"]}
        if pred:
            n = max(dm["trace_supplied"], 1)
            row["predictor_stats"] = {"predictions": dm["trace_supplied"], "head_top_frac": round(dm["head_top"] / n, 4),
                                      "head_active_frac": round(dm["head_active"] / n, 4),
                                      "head_inactive_frac": round(dm["head_inactive"] / n, 4),
                                      "issued": dm["issued"], "cancelled": dm["cancelled"]}
        res[name] = row
        st.close()
    out.update(res)
    return out


def c2_tier(capi, torch, hbm, pcie, cpu):
    """The headline workload with the HBM expert tier (moeb_set_expert_sources;
    SURVEY §8(f) rank 4): misses uploaded from a device-resident copy of the
    pool (LocalTier: this GPU's HBM — on one GPU the stand-in for a peer GPU's
    HBM over NVLink 5) instead of pinned host memory. A device tier runs the
    uploads in serial mode, so the host-pool serial run is the like-for-like
    comparison; decisions are identical in all three."""
    from paper_2508_18983_b200.tier import LocalTier
    cfg, model = split(DSV2)
    cfg_d = dict(cfg, num_layers=26, batch=1, slots=16, alpha=0.25, seed=7)
    T, K = 64, 48
    out = {"workload": "DeepSeek-V2-Lite 26 L, batch 1, cache 16/64, trace-driven, CE+ER+Pre+BA"}
    # the stack that creates the pinned pool runs first and is not reported:
    # the first decode from a freshly pinned 28.8 GB pool measured up to 9.9
    # vs 7.3-7.4 ms/token on later stacks sharing it
    row, pool, _ = run_case(capi, torch, cfg_d, model, T, K, hbm, pcie)
    row, st, _ = run_case(capi, torch, cfg_d, model, T, K, hbm, pcie, pool=pool)
    st.close()
    out["host_pool_pipelined"] = row
    os.environ["MOEB_SERIAL"] = "1"
    row, st, _ = run_case(capi, torch, cfg_d, model, T, K, hbm, pcie, pool=pool)
    st.close()
    out["host_pool_serial"] = row
    os.environ.pop("MOEB_SERIAL")
    tiers = []
    row, st, _ = run_case(capi, torch, cfg_d, model, T, K, hbm, pcie, pool=pool,
                          setup=lambda s: tiers.append(LocalTier(torch, s, 26 * 64)))
    st.close()
    tiers.clear()
    pool.close()
    up = row["path_roofline"]["pcie_mb_per_step"] * 1e6
    b_hbm = row["path_roofline"]["hbm_mb_per_step"] * 1e6
    # the tier copies read and write HBM: the bound is HBM, not PCIe
    t_roof = (b_hbm + 2 * up) / (hbm * 1e9) * 1e3
    row["path_roofline"] = {"t_roof_ms": round(t_roof, 4), "frac": round(t_roof / row["ms_per_token"], 4),
                            "hbm_mb_per_step": round(b_hbm / 1e6, 1), "tier_mb_per_step": round(up / 1e6, 1),
                            "bound": "hbm"}
    # a peer GPU's HBM over NVLink 5 (900 GB/s per direction) instead of this GPU's
    row["nvlink5_projection_ms"] = round(max(b_hbm / (hbm * 1e9), up / 900e9) * 1e3, 4)
    out["device_tier_serial"] = row
    return out


def c5(capi, torch, hbm, pcie, cpu):
    from paper_2508_18983_b200 import partition
    out = {"workload": "64 DeepSeek-V2-Lite requests x 16 tokens, stream-partitioned, cache 16/64, 1 GPU", "batch": {}}
    pools = partition.NodePools(None, 0, "cfg")
    for B in (1, 2, 4, 8, 16, 32):
        out["batch"][f"B{B}"] = bench.c5_partitioned(capi, partition, torch, None, pools, 1, 0, 0, B)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2P,C2T,C3,C4,C5")
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    from paper_2508_18983_b200 import partition
    partition.bind_to_device_node(0)  # pinned pools first-touched on the GPU's NUMA node
    import torch
    from paper_2508_18983_b200 import capi
    torch.cuda.set_device(0)
    hbm, _ = bench.peaks()
    pcie = bench.measure_pcie_gbs(torch)
    res = {"hbm_peak_gbs": hbm, "pcie_peak_gbs": round(pcie, 2), "gpu": torch.cuda.get_device_name(0)}
    for name in args.only.split(","):
        t0 = time.time()
        res[name] = {"C1": c1, "C2P": c2_predictor, "C2T": c2_tier, "C3": c3, "C4": c4, "C5": c5}[name](capi, torch, hbm, pcie,
                                                                                     not args.no_cpu)
        res[name]["wall_s"] = round(time.time() - t0, 1)
        print(f"{name} done in {res[name]['wall_s']} s", file=sys.stderr, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
