#!/usr/bin/env python3
"""Bench: MoE decode ms/token + expert cache hit rate, DeepSeek-V2-Lite shape.

Workload (BASELINE.json configs[1]): the 26-layer DeepSeek-V2-Lite MoE stack
(64 routed experts top-6 + 2 shared, d=2048, ffn=1408), batch-1 decode of a
512-token synthetic stream, expert cache capped at 25% (16 of 64 experts per
layer), full scheduler stages CE+ER+Pre+BA at alpha=0.25 — plus the same
stream with substitution off (ER off) as an ablation.

A "step" is one decoded token through all 26 layers: per layer the router
gate kernel, the device decision kernel (routing / substitution / cache /
prefetch / balance, bit-exact vs the reference), and the persistent grouped
SwiGLU FFN kernel; expert misses are uploaded from pinned host memory over
PCIe on the copy stream while resident experts compute.

Data: synthetic. Router logits are ln(s) of the reference's generate_trace
(trace.cpp:106, seed 7 + rank) so the softmax reproduces the reference's
skewed, temporally persistent routing; hidden states are an AR(1) stream;
weights are counter-based random (uniform +-sqrt(3/fan_in), bf16).

Timed region: W warm-up tokens (untimed, positions 0..W-1), then exactly K
tokens (positions W..W+K-1), bracketed by barrier + synchronize, CUDA events
on the stack's stream, max over ranks. Every step streams ~140 MB of expert
weights from HBM and hundreds of MB over PCIe, far above the 126 MB L2, so no
L2 flush is needed ("l2": "inputs > L2").

--impl reference: the reference's CPU path on this host (decisions by the
reference library compiled from /root/reference into oracle/_ref, layer
arithmetic by the CPU fp32 port oracle/cpu_moe.c over all host threads).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# DeepSeek-V2-Lite MoE stack (configs[1]); CE+ER+Pre+BA, alpha 0.25, c = 25% of E
CFG = dict(num_layers=26, experts=64, top_k=6, batch=1, alpha=0.25, slots=16, window=16, seed=7,
           ce=1, er=1, pre=1, ba=1)
MODEL = dict(d_model=2048, ffn=1408, shared_ffn=2816, shared_gate=0, renormalize=0, routed_scale=1.0)
TOKENS = 512
FFN_KERNEL_B1 = "ffn_splitk_kernel"  # the batch-1 FFN (csrc/ffn_splitk.cuh) the roofline line measures


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 4 + i and r[4 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ar1_hidden(T, B, d, seed):
    rng = np.random.default_rng(seed)
    x = np.zeros((T, B, d), dtype=np.float32)
    prev = rng.standard_normal((B, d)).astype(np.float32)
    for t in range(T):
        prev = 0.9 * prev + np.float32(np.sqrt(0.19)) * rng.standard_normal((B, d)).astype(np.float32)
        x[t] = prev
    return x


def divergence(y_sub, y_exact, x_in):
    """Substituted (ER on) vs exact (ER off) decode outputs on the same tokens.

    Per token: relative L2 and max-relative error of the final hidden state,
    and relative L2 of the MoE stack's contribution (final hidden - input).
    """
    T = y_sub.shape[0]
    a = y_sub.reshape(T, -1).astype(np.float64)
    b = y_exact.reshape(T, -1).astype(np.float64)
    x = x_in.reshape(T, -1).astype(np.float64)
    diff = np.linalg.norm(a - b, axis=1)
    rel = diff / np.maximum(np.linalg.norm(b, axis=1), 1e-30)
    mrel = np.abs(a - b).max(axis=1) / np.maximum(np.abs(b).max(axis=1), 1e-30)
    drel = diff / np.maximum(np.linalg.norm(b - x, axis=1), 1e-30)
    return {"tokens": int(T), "hidden_rel_l2_mean": round(float(rel.mean()), 5),
            "hidden_rel_l2_max": round(float(rel.max()), 5), "hidden_max_rel_mean": round(float(mrel.mean()), 5),
            "moe_delta_rel_l2_mean": round(float(drel.mean()), 5), "moe_delta_rel_l2_max": round(float(drel.max()), 5),
            "identical_tokens": int((diff == 0).sum())}


def timeline_summary(tl):
    """Per layer-step averages (us) from the device-clock timeline rows
    (moeb_get_timeline): decide entry->publish/end, FFN duration, gaps."""
    tl = tl.astype(np.int64)
    up = tl[:, 1] != 0
    r = lambda v: round(float(np.mean(v)) / 1e3, 2) if len(v) else None
    spec = tl[:, 6] != 0
    # FFN busy span: from the speculative plan (or the final plan) to the end
    start = np.where(spec, tl[:, 6], tl[:, 0])
    return {"decide_to_publish_us": r(tl[:, 4] - tl[:, 3]), "decide_us": r(tl[:, 5] - tl[:, 3]),
            "ffn_us": r((tl[:, 2] - tl[:, 0])[~up]) if (~up).any() else None,
            "ffn_span_us": r((tl[:, 2] - start)[~up]) if (~up).any() else None,
            "ffn_overlap_with_decide_us": r((tl[:, 5] - tl[:, 6])[spec]) if spec.any() else None,
            "ffn_tail_after_last_upload_us": r((tl[:, 2] - tl[:, 1])[up]) if up.any() else None,
            "gap_decide_to_ffn_us": r(tl[:, 0] - tl[:, 5]), "gap_ffn_to_next_decide_us": r(tl[1:, 3] - tl[:-1, 2]),
            "layer_period_us": r(tl[1:, 3] - tl[:-1, 3]), "layer_steps_with_uploads": int(up.sum()),
            "layer_steps": int(len(tl))}


def measure_pcie_gbs(torch):
    """Pinned H2D copy-engine bandwidth (the PCIe roofline): four back-to-back
    256 MB copies per sample, best of 5."""
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best = 1e9
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(4):
                d.copy_(h, non_blocking=True)
            b.record(s)
            b.synchronize()
            best = min(best, a.elapsed_time(b) / 4)
    del h, d
    return n / best / 1e6


def batched_section(capi, torch, local, hbm_peak, batches=(8, 32), n_warm=8, n_timed=32):
    """Config C5 (independent decode streams, DeepSeek-V2-Lite shape) at
    batch B on one GPU: the batched tensor-core FFN (ffn_umma.cuh). Per B:
    ms/step and tokens/s with the 16/64 cache (PCIe uploads), and the FFN
    kernel's HBM roofline on the all-resident configuration (CUDA events
    around every FFN launch, algorithmic bytes = every selected expert's
    weights once)."""
    L, E, d = CFG["num_layers"], CFG["experts"], MODEL["d_model"]
    T = n_warm + n_timed
    out = {}
    pool = None  # the UMMA-tiled host pool, generated once, shared by every batched stack
    for B in batches:
        scores = capi.generate_trace(L, E, B, T, 7)
        logits = capi.trace_logits(scores)
        x = torch.from_numpy(ar1_hidden(T, B, d, 7)).to(torch.bfloat16).cuda()
        y = torch.empty((B, d), dtype=torch.bfloat16, device="cuda")
        row = {}
        # cache 16/64; all-resident as it runs (PDL chain, speculative
        # gate_up); all-resident with CUDA events around every FFN launch
        for mode in ("cache", "allhit", "allhit_events"):
            allhit = mode != "cache"
            cfg = capi.Config.make(**dict(CFG, batch=B, slots=E if allhit else CFG["slots"]))
            kw = dict(time_kernels=mode == "allhit_events")
            # the event pass times the FFN standalone: no speculative phase
            # (events serialise the launches, nothing to overlap with)
            if mode == "allhit_events":
                os.environ["MOEB_NO_SPEC"] = "1"
            else:
                os.environ.pop("MOEB_NO_SPEC", None)
            if pool is not None:
                kw["weights_host"] = pool
            st = capi.Stack(cfg, weight_seed=7, device=local, **kw, **MODEL)
            if pool is None:
                pool = (st.host_pool()[0], st)
            st.set_logits_trace(logits, T)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for i in range(n_warm):
                    st.step(x[i].data_ptr(), y.data_ptr(), B, stream=s.cuda_stream)
                st.sync()
                m0 = st.metrics()
                st.reset_kernel_stats()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for i in range(n_warm, T):
                    st.step(x[i].data_ptr(), y.data_ptr(), B, stream=s.cuda_stream)
                if not allhit:
                    st.sync()  # every upload the timed steps published has landed
                e1.record(s)
                e1.synchronize()
                st.sync()
            ms = e0.elapsed_time(e1) / n_timed
            m1 = st.metrics()
            if mode == "allhit":
                row["all_resident"] = {"ms_per_step": round(ms, 4), "tokens_per_s": round(B * 1e3 / ms, 1)}
            elif allhit:
                k = st.kernel_stats()
                gbs = k["ffn_bytes"] / (k["ffn_ms"] * 1e-3) / 1e9
                row["all_resident"].update({"ms_per_step_events": round(ms, 4),
                                       "ffn_us_per_launch": round(k["ffn_ms"] * 1e3 / max(k["ffn_launches"], 1), 2),
                                       "ffn_mb_per_launch": round(k["ffn_bytes"] / max(k["ffn_launches"], 1) / 1e6, 1),
                                       "ffn_achieved_gbs": round(gbs, 1), "ffn_frac": round(gbs / hbm_peak, 4)})
            else:
                sel = m1["selections"] - m0["selections"]
                row["cache_16_of_64"] = {"ms_per_step": round(ms, 4), "tokens_per_s": round(B * 1e3 / ms, 1),
                                         "hit_rate": round((m1["hits"] - m0["hits"]) / max(sel, 1), 4)}
            if st is not pool[1]:
                st.close()
        out[f"B{B}"] = row
    os.environ.pop("MOEB_NO_SPEC", None)
    pool[1].close()
    out["note"] = ("config C5 shape, one GPU, steps " + str(n_timed) + " after " + str(n_warm) +
                   " warm-up; FFN = tcgen05 kernel (UMMA-tiled experts); ms_per_step = the PDL "
                   "pipeline as it runs; ffn_* from a second all-resident pass with CUDA events around "
                   "every FFN launch (standalone kernel, launch latency included, no overlap)")
    return out


def c5_partitioned(capi, partition, torch, dist, pools, world, rank, local, B, tokens=16, n_requests=64,
                   n_warm=3):
    """Config C5 as specified: n_requests independent DeepSeek-V2-Lite decode
    streams at batch B, stream-partitioned across the world's GPUs
    (partition.partition: contiguous blocks of batch groups), each GPU with
    its own 16/64 expert cache, copy stream and PCIe link, no collective on
    the data path. Every rank decodes its groups back to back; the whole-job
    time is the max over ranks. Collective over all ranks (setup + timing)."""
    L, E, d = CFG["num_layers"], CFG["experts"], MODEL["d_model"]
    groups = partition.partition(n_requests, B, world, rank)
    scores = partition.sub_stream(capi, L, E, B, tokens, groups)
    T = scores.shape[0]
    cfg = capi.Config.make(**dict(CFG, batch=B))
    pool_bytes = L * E * 3 * MODEL["ffn"] * d * 2
    st = pools.stack(capi, cfg, "rows" if B == 1 else "tiled", pool_bytes, weight_seed=7, device=local, **MODEL)
    st.set_logits_trace(capi.trace_logits(scores), T)
    x = torch.from_numpy(np.concatenate([ar1_hidden(tokens, B, d, partition.group_seed(g)) for g in groups])) \
        .to(torch.bfloat16).cuda()
    y = torch.empty((B, d), dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(n_warm):  # first launches, then back to the initial state
            st.step(x[i].data_ptr(), y.data_ptr(), B, stream=s.cuda_stream)
        st.sync()
        st.reset()
        io0 = st.io_stats()  # the warm-up's uploads are not part of the timed job
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for i in range(T):
            st.step(x[i].data_ptr(), y.data_ptr(), B, stream=s.cuda_stream)
        st.sync()  # every upload the timed steps published has landed (they are counted)
        e1.record(s)
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    m = st.metrics()
    io = {k: v - io0.get(k, 0) if isinstance(v, (int, float)) else v for k, v in st.io_stats().items()}
    st.close()
    # this GPU's link for the path roofline: the probe, or the run's own copy rate if higher
    pcie = max(measure_pcie_gbs(torch), io["h2d_bytes"] / max(io["copy_ms"], 1e-9) / 1e6)
    # the uploads the decisions call for (speculative chunks excluded)
    eb = 3 * MODEL["ffn"] * d * 2
    up = float(io["h2d_bytes"] - io["spec_bytes"] + io["spec_promoted"] * eb)
    mine = torch.tensor([ms, float(T * B), float(m["hits"]), float(m["selections"]), up,
                         up / (pcie * 1e9) * 1e3], dtype=torch.float64)
    if world > 1:
        allv = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allv, mine)
    else:
        allv = [mine]
    allv = torch.stack(allv).numpy()
    t_max = float(allv[:, 0].max())
    toks = float(allv[:, 1].sum())
    t_roof = float(allv[:, 5].max())  # the slowest link's upload time (PCIe-bound)
    return {"batch": B, "requests": n_requests, "tokens_per_request": tokens, "gpus": world,
            "groups_per_gpu": len(groups), "whole_job_ms": round(t_max, 2),
            "path_roofline": {"t_roof_ms": round(t_roof, 2), "frac": round(t_roof / t_max, 4), "bound": "pcie"},
            "tokens_per_s": round(toks / (t_max * 1e-3), 1),
            "per_gpu_tokens_per_s": [round(float(r[1] / (r[0] * 1e-3)), 1) for r in allv],
            "hit_rate": round(float(allv[:, 2].sum() / max(allv[:, 3].sum(), 1)), 4),
            "pcie_gb_per_gpu": [round(float(r[4]) / 1e9, 3) for r in allv],
            "ms_per_token_whole_job": round(t_max / toks, 4)}


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2508_18983_b200 import capi, partition

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # MOEB_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo (exercises the
    # multi-rank path on a one-GPU box; not a scaling measurement)
    share_gpu = os.environ.get("MOEB_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local = 0
    torch.cuda.set_device(local)
    # no NCCL anywhere: the data path has no collective (north star); gloo
    # carries the setup exchange, the barriers and the max/sum of timings
    coll_dev = "cpu"
    if world > 1:
        dist.init_process_group("gloo")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    W, K = args.warmup, args.steps
    # the whole 512-token stream of configs[1] is decoded; the timed tokens
    # are its last K (so the cache is in its steady state), everything
    # before them is untimed warm-up (>= W tokens)
    T = max(TOKENS, W + K)
    W = T - K
    L, E, B, d = CFG["num_layers"], CFG["experts"], CFG["batch"], MODEL["d_model"]
    seed = 7 + rank  # independent decode stream per GPU (stream partitioning, no collective)
    scores = capi.generate_trace(L, E, B, T, seed)
    logits = capi.trace_logits(scores)
    x_host = ar1_hidden(T, B, d, seed)
    x_dev = torch.from_numpy(x_host).to(torch.bfloat16).cuda()
    x_pin = x_dev.cpu().pin_memory()
    y_dev = torch.empty((B, d), dtype=torch.bfloat16, device="cuda")
    y_pin = torch.empty((T, B, d), dtype=torch.bfloat16).pin_memory()

    cfg = capi.Config.make(**CFG)
    t0 = time.time()
    # no per-kernel CUDA events in the timed stack (they would serialise the
    # programmatic dependent launches); the per-kernel split comes from the
    # device-clock timeline (globaltimer stamps written by the kernels)
    # pinned host pools: one replica per NUMA node of GPUs (28.8 GB each),
    # filled by the node's first rank and mapped by the others
    pools = partition.NodePools(dist if world > 1 else None, local,
                                os.environ.get("TORCHELASTIC_RUN_ID", "run") + "_" + os.environ.get("MASTER_PORT", "0"))
    pool_bytes = L * E * 3 * MODEL["ffn"] * d * 2
    stack = pools.stack(capi, cfg, "rows", pool_bytes, weight_seed=7, trace_timeline=True, device=local, **MODEL)
    create_s = time.time() - t0
    stack.set_logits_trace(logits, T)
    # a torch-owned stream for the stack's work: pinned-buffer copies recorded
    # on it stay valid after the stack (and its internal streams) is destroyed
    s = torch.cuda.Stream()
    s_ptr = s.cuda_stream

    def run_steps(lo, hi, e2e=False):
        for i in range(lo, hi):
            if e2e:
                xi = x_dev[i]
                xi.copy_(x_pin[i], non_blocking=True)  # H2D of this step's input
                stack.step(xi.data_ptr(), y_dev.data_ptr(), B, stream=s_ptr)
                y_pin[i].copy_(y_dev, non_blocking=True)  # D2H of this step's output
            else:
                stack.step(x_dev[i].data_ptr(), y_dev.data_ptr(), B, stream=s_ptr)

    # ---- device-resident inputs (value)
    with torch.cuda.stream(s):
        run_steps(0, W)
        stack.sync()
        m0 = stack.metrics()
        stack.reset_kernel_stats()
        barrier()
        clocks = ClockSampler(local)
        clocks.start()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(s)
        run_steps(W, T)
        ev1.record(s)
        ev1.synchronize()
        stack.sync()
        barrier()
        clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    m1 = stack.metrics()
    io = stack.io_stats()
    ks = stack.kernel_stats()
    tl_main = timeline_summary(stack.timeline()[-K * L:])
    ms_max = max_over_ranks(ms)

    # ---- end to end through the C-ABI with host buffers (e2e)
    stack.reset()
    with torch.cuda.stream(s):
        run_steps(0, W, e2e=True)
        stack.sync()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        run_steps(W, T, e2e=True)
        e1.record(s)
        e1.synchronize()
        stack.sync()
        barrier()
    e2e_ms_max = max_over_ranks(e0.elapsed_time(e1))

    # ---- substitution off (ER off), same stream and weights (ablation)
    abl = None
    if not args.no_ablation:
        cfg2 = capi.Config.make(**dict(CFG, er=0))
        pool_ptr, _ = stack.host_pool()
        st2 = capi.Stack(cfg2, weight_seed=7, device=local, weights_host=(pool_ptr, stack), **MODEL)
        st2.set_logits_trace(logits, T)
        s2 = torch.cuda.Stream()
        s2p = s2.cuda_stream
        y_off = torch.empty((T, B, d), dtype=torch.bfloat16, device="cuda")
        with torch.cuda.stream(s2):
            for i in range(W):
                st2.step(x_dev[i].data_ptr(), y_off[i].data_ptr(), B, stream=s2p)
            st2.sync()
            a0m = st2.metrics()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(s2)
            for i in range(W, T):
                st2.step(x_dev[i].data_ptr(), y_off[i].data_ptr(), B, stream=s2p)
            a1.record(s2)
            a1.synchronize()
            st2.sync()
        a1m = st2.metrics()
        sel = a1m["selections"] - a0m["selections"]
        abl = {"er_off": {"ms_per_token": round(a0.elapsed_time(a1) / K, 4),
                          "hit_rate": round((a1m["hits"] - a0m["hits"]) / max(sel, 1), 4),
                          "demand_loads": a1m["demand_loads"] - a0m["demand_loads"],
                          "streamed": a1m["cpu_computed"] - a0m["cpu_computed"]}}
        st2.close()
        # substituted-vs-exact output divergence: the ER-on outputs of the e2e
        # run (same stream, same initial cache) against these ER-off outputs
        abl["divergence"] = divergence(y_pin[W:T].float().numpy(), y_off[W:T].float().cpu().numpy(),
                                       x_dev[W:T].float().cpu().numpy())
        # the same stream WITH speculative uploads (opt-in experiment, identical decisions)
        os.environ["MOEB_SPEC_UPLOAD"] = "1"
        try:
            st4 = capi.Stack(cfg, weight_seed=7, device=local, weights_host=(pool_ptr, stack), **MODEL)
        finally:
            del os.environ["MOEB_SPEC_UPLOAD"]
        st4.set_logits_trace(logits, T)
        with torch.cuda.stream(s2):
            for i in range(W):
                st4.step(x_dev[i].data_ptr(), y_dev.data_ptr(), B, stream=s2p)
            st4.sync()
            b0m = st4.metrics()
            a0.record(s2)
            for i in range(W, T):
                st4.step(x_dev[i].data_ptr(), y_dev.data_ptr(), B, stream=s2p)
            a1.record(s2)
            a1.synchronize()
            st4.sync()
        b1m = st4.metrics()
        io4 = st4.io_stats()
        abl["spec_upload_on"] = {"ms_per_token": round(a0.elapsed_time(a1) / K, 4),
                                 "jobs": io4["spec_jobs"], "used": io4["spec_promoted"],
                                 "same_decisions": (b1m["hits"] - b0m["hits"]) == (m1["hits"] - m0["hits"]) and
                                 (b1m["demand_loads"] - b0m["demand_loads"]) == (m1["demand_loads"] - m0["demand_loads"])}
        st4.close()

    # ---- FFN kernel roofline on the all-resident configuration (no uploads)
    hbm_peak, peak_kind = peaks()
    cfg3 = capi.Config.make(**dict(CFG, slots=E))
    pool_ptr, _ = stack.host_pool()
    n3 = min(64, T)

    def allhit_pass(**kw):
        st3 = capi.Stack(cfg3, weight_seed=7, device=local, weights_host=(pool_ptr, stack), **kw, **MODEL)
        st3.set_logits_trace(logits, T)
        s3 = torch.cuda.Stream()
        s3p = s3.cuda_stream
        with torch.cuda.stream(s3):
            for i in range(8):
                st3.step(x_dev[i].data_ptr(), y_dev.data_ptr(), B, stream=s3p)
            st3.sync()
            st3.reset_kernel_stats()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(s3)
            for i in range(8, 8 + n3):
                st3.step(x_dev[i % T].data_ptr(), y_dev.data_ptr(), B, stream=s3p)
            a1.record(s3)
            a1.synchronize()
            st3.sync()
        out = (a0.elapsed_time(a1) / n3, st3.kernel_stats(), st3.timeline()[-n3 * L:] if kw.get("trace_timeline") else None)
        st3.close()
        return out

    # (1) CUDA events around every FFN launch on its stream: the roofline's
    # conservative per-launch duration. Events stop the launches from
    # overlapping (no PDL), so the FFN runs as a standalone kernel here: the
    # speculative start is switched off for this pass (it would only add a
    # second gate_up phase with nothing to overlap) and the duration includes
    # the launch latency.
    os.environ["MOEB_NO_SPEC"] = "1"
    try:
        _, k3, _ = allhit_pass(time_kernels=True)
    finally:
        del os.environ["MOEB_NO_SPEC"]
    # (2) the same work as it runs in the stack (no events): ms/token and the
    # device-clock FFN duration
    allhit_ms_token, _, tl3 = allhit_pass(trace_timeline=True)
    tl_hit = timeline_summary(tl3)
    ffn_gbs = k3["ffn_bytes"] / (k3["ffn_ms"] * 1e-3) / 1e9
    per_launch_bytes = k3["ffn_bytes"] / max(k3["ffn_launches"], 1)
    # DRAM bytes per launch of the SAME kernel from a committed ncu --set full
    # capture of this configuration (null if the capture is of another kernel)
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(REPO, "profiles", "ncu_ffn_traffic.json")) as f:
            tj = json.load(f)
        if FFN_KERNEL_B1 in tj.get("kernel", ""):
            traffic, traffic_src = tj.get("dram_bytes_per_launch"), tj.get("source")
    except Exception:
        pass

    # ---- path roofline: T_roof = max(B_hbm / BW_hbm, B_pcie / BW_pcie) per token
    # the copy engine's own rate during the timed run is a floor for the peak
    # (a single 256 MB probe can land on a momentarily slower link)
    pcie_probe = measure_pcie_gbs(torch)
    pcie_run = io["h2d_bytes"] / max(io["copy_ms"], 1e-9) / 1e6
    pcie_peak = max(pcie_probe, pcie_run)
    tokens = K
    b_hbm = (ks["ffn_bytes"] + ks["route_bytes"]) / tokens
    # algorithmic PCIe bytes: the uploads the decisions call for (each expert
    # once); speculative chunks that went unused are not part of the roofline
    eb = 3 * MODEL["ffn"] * d * 2
    b_pcie = (io["h2d_bytes"] - io["spec_bytes"] + io["spec_promoted"] * eb) / tokens
    t_roof = max(b_hbm / (hbm_peak * 1e9), b_pcie / (pcie_peak * 1e9)) * 1e3
    ms_tok = ms / K
    sel = m1["selections"] - m0["selections"]
    hit = (m1["hits"] - m0["hits"]) / max(sel, 1)

    total_tokens = sum_over_ranks(float(K))
    value = ms_max / (total_tokens / world) / world  # whole-job ms per token across all GPUs
    result = {
        "metric": "MoE decode ms/token + expert cache hit rate, DeepSeek-V2-Lite shape",
        "value": round(value, 4),
        "unit": "ms/token",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max / K, 4),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16 weights, fp32 accumulate; fp64 decisions",
        "data": "synthetic: reference generate_trace router logits (seed 7+rank), AR(1) hidden states, "
                "counter-based random bf16 weights",
        "config": {"workload": f"DeepSeek-V2-Lite 26-layer MoE stack, batch-1 decode of a {T}-token stream "
                               f"(timed: its last {K} tokens), cache 16/64 experts per layer, CE+ER+Pre+BA "
                               "alpha=0.25",
                   "stream_tokens": T, "untimed_tokens_before_window": W, "layers": L, "experts": E, "top_k": CFG["top_k"], "shared_ffn": MODEL["shared_ffn"],
                   "d_model": d, "ffn": MODEL["ffn"], "global_batch": B * world, "tokens_per_gpu_timed": K,
                   "slots_per_layer": CFG["slots"], "parallelism": f"stream-partitioned x{world} (no collective)",
                   "l2": "inputs > L2 (>=140 MB weights per step)"},
        "hit_rate": round(hit, 4),
        "metrics_timed": {"demand_loads": m1["demand_loads"] - m0["demand_loads"],
                          "streamed_ba": m1["cpu_computed"] - m0["cpu_computed"],
                          "prefetch_loads": m1["prefetch_loads"] - m0["prefetch_loads"],
                          "substitutions": m1["substitutions"] - m0["substitutions"],
                          "substitution_ratio": round((m1["substitutions"] - m0["substitutions"]) /
                                                      max(1, (m1["substitutions"] - m0["substitutions"]) +
                                                          (m1["low_score_kept"] - m0["low_score_kept"])), 4)},
        "e2e": {"value": round(e2e_ms_max / K / world, 4), "unit": "ms/token", "h2d_bytes_per_step": B * d * 2,
                "d2h_bytes_per_step": B * d * 2},
        "roofline": {"bound": "hbm", "kernel": f"{FFN_KERNEL_B1} (all-resident pass, no uploads)",
                     "achieved": round(ffn_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(ffn_gbs / hbm_peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "device_clock_span_us": tl_hit["ffn_span_us"],
                     "device_clock_achieved": round(per_launch_bytes / (tl_hit["ffn_span_us"] * 1e-6) / 1e9, 1),
                     "device_clock_frac": round(per_launch_bytes / (tl_hit["ffn_span_us"] * 1e-6) / 1e9 / hbm_peak, 4),
                     "algorithmic_bytes_per_launch": int(per_launch_bytes), "peak_source": peak_kind,
                     "allhit_ms_per_token": round(allhit_ms_token, 4)},
        "path_roofline": {"t_roof_ms": round(t_roof, 4), "t_measured_ms": round(ms_tok, 4),
                          "frac": round(t_roof / ms_tok, 4), "hbm_bytes_per_token": int(b_hbm),
                          "pcie_bytes_per_token": int(b_pcie),
                          "pcie_bytes_moved_per_token": int(io["h2d_bytes"] / tokens),
                          "pcie_peak_gbs": round(pcie_peak, 2),
                          "pcie_probe_gbs": round(pcie_probe, 2),
                          "pcie_achieved_gbs_copy_stream": round(io["h2d_bytes"] / max(io["copy_ms"], 1e-9) / 1e6, 2),
                          "pcie_busy_frac": round(io["copy_ms"] / ms, 4),
                          "bound": "pcie" if b_pcie / pcie_peak > b_hbm / hbm_peak else "hbm"},
        "layer_us_device_clock": {"timed_run": tl_main, "all_resident": tl_hit},
        "allhit_ffn_event_us": round(k3["ffn_ms"] * 1e3 / max(k3["ffn_launches"], 1), 2),
        "gpu_launches": int(2 * L * K),
        "clocks": clk,
        "create_s": round(create_s, 2),
    }
    if abl:
        result["ablation"] = abl
    if world == 1 and not args.no_prefill:
        result["prefill"] = prefill_section(torch, stack, d, pcie_peak, hbm_peak)
    if not args.no_c5:
        # C5: 64 requests stream-partitioned over the world's GPUs at the
        # largest batch the partition allows (B <= 64 / G, <= 32)
        stack.close()
        stack = None
        Bc5 = min(32, 64 // world)
        result["c5_partitioned"] = c5_partitioned(capi, partition, torch, dist, pools, world, rank, local, Bc5)
    if rank == 0 and world == 1 and not args.no_batched:
        if stack is not None:
            stack.close()
        stack = None
        result["batched_c5"] = batched_section(capi, torch, local, hbm_peak)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(scores, x_host, args.cpu_sample_tokens)
    torch.cuda.synchronize()
    del x_pin, y_pin
    if stack is not None:
        stack.close()
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def prefill_section(torch, stack, d, pcie_peak, hbm_peak, N=512, reps=2):
    """Prefill (moeb_prefill) of an N-token prompt on the bench's own stack
    (batch 1, cache 16/64: experts re-tiled per layer, the 48 non-resident
    experts of every layer uploaded while the previous layer computes): TTFT
    with CUDA events on the stream, against the PCIe path roofline."""
    g = torch.Generator().manual_seed(11)
    x = (torch.randn(N, d, generator=g) * 2).to(torch.bfloat16).cuda()
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    stack.prefill(x.data_ptr(), y.data_ptr(), N, stream=s.cuda_stream)  # warm-up: buffers
    torch.cuda.synchronize()
    ts, up = [], 0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        up = stack.prefill(x.data_ptr(), y.data_ptr(), N, stream=s.cuda_stream)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    L, E = CFG["num_layers"], CFG["experts"]
    wbytes = L * (E * d * 2 + 3 * MODEL["shared_ffn"] * d * 2) + L * E * 3 * MODEL["ffn"] * d * 2
    # the PCIe peak: the bench's probe, or this run's own large-copy rate if higher
    bw = max(pcie_peak, up / (ms * 1e-3) / 1e9)
    t_roof = max(up / (bw * 1e9), wbytes / (hbm_peak * 1e9)) * 1e3
    return {"tokens": N, "ttft_ms": round(ms, 2), "tokens_per_s": round(N / (ms * 1e-3), 1),
            "upload_gb": round(up / 1e9, 3), "pcie_achieved_gbs": round(up / (ms * 1e-3) / 1e9, 2),
            "path_roofline": {"t_roof_ms": round(t_roof, 2), "frac": round(t_roof / ms, 4), "bound": "pcie",
                              "pcie_peak_gbs": round(bw, 2)},
            "note": "plain top-k routing, grouped tcgen05 GEMM; tools/bench_prefill.py for the all-resident "
                    "(HBM / tensor-bound) numbers"}


# ----------------------------------------------------------------- CPU path

def cpu_path(scores, x_host, n_tokens, nthreads, cfg_d=None, model_d=None):
    """The reference CPU path: reference-library decisions + CPU fp32 layer arithmetic.

    Decisions: the reference's simulate() (oracle/_ref, compiled from
    /root/reference) when present, else the oracle's C port, over all tokens
    (single-threaded, as the reference runs); the per-token selections for
    the arithmetic come from the oracle's per-step records (== the reference's
    decisions: tests/test_golden.py). Arithmetic: oracle/cpu_moe.c (fp32 over
    bf16 weights in host RAM, persistent pool over every host thread, AVX2)
    for the last n_tokens tokens, every token of the batch separately.
    Returns (ms_per_token, kind, cores, sample, host_weight_gbs).
    """
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import pyoracle as po

    cfg_d = cfg_d or CFG
    model_d = model_d or MODEL
    L, E, B = cfg_d["num_layers"], cfg_d["experts"], cfg_d["batch"]
    d, F, S = model_d["d_model"], model_d["ffn"], model_d["shared_ffn"]
    sg, renorm, rscale = model_d.get("shared_gate", 0), model_d.get("renormalize", 0), model_d.get("routed_scale", 1.0)
    T = scores.shape[0]
    cfg = po.SimCfg(**{k: v for k, v in cfg_d.items()})
    use_ref = po.ref() is not None
    if use_ref:
        dec_s = po.ref_simulate_seconds(cfg, scores)  # simulate() alone, timed inside the library
    else:
        t0 = time.perf_counter()
        po.simulate(cfg, scores, timeline=False)
        dec_s = time.perf_counter() - t0
    dec_ms_token = dec_s * 1e3 / T
    steps = po.simulate(cfg, scores, steps=True, timeline=False)["steps"]
    sel_of = {(r["it"], r["layer"]): [t["sel"] for t in r["tok"]] for r in steps}

    cm = C.CDLL(os.path.join(REPO, "oracle", "libcpumoe.so"))
    cm.cpu_synth.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p, C.c_int]
    cm.cpu_moe_layer.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_int]
    cm.cpu_bytes_touched.restype = C.c_uint64
    seed = 7

    def tid(l, e, m):
        return (l << 20) | (e << 4) | m

    cache = {}

    def tensor(key, tensor_id, n, fan_in):
        if key not in cache:
            a = np.empty(n, dtype=np.uint16)
            cm.cpu_synth(seed, tensor_id, n, fan_in, a.ctypes.data, nthreads)
            cache[key] = a
        return cache[key]

    def expert(l, e):
        key = ("e", l, e)
        if key not in cache:
            a = np.empty(3 * F * d, dtype=np.uint16)
            for m in range(3):
                cm.cpu_synth(seed, tid(l, e, m), F * d, d if m < 2 else F, a[m * F * d:].ctypes.data, nthreads)
            cache[key] = a
        return cache[key]

    # weights in host RAM before timing (the CPU path has no PCIe)
    sample = list(range(T - n_tokens, T))
    for l in range(L):
        tensor(("r", l), (l << 20) | (0xFFFF << 4), E * d, d)
        if sg:
            tensor(("g", l), (l << 20) | (0xFFFD << 4), d, d)
        if S:
            sh = np.empty(3 * S * d, dtype=np.uint16)
            for m in range(3):
                cm.cpu_synth(seed, (l << 20) | (0xFFFE << 4) | m, S * d, d if m < 2 else S,
                             sh[m * S * d:].ctypes.data, nthreads)
            cache[("s", l)] = sh
        for it in sample:
            for sel in sel_of[(it, l)]:
                for e in sel:
                    expert(l, e)
    logits = np.zeros(E, dtype=np.float32)
    y = np.zeros(d, dtype=np.float32)
    cm.cpu_bytes_touched()
    t0 = time.perf_counter()
    for it in sample:
        for t in range(B):
            x = np.ascontiguousarray(x_host[it, t]).astype(np.float32)
            xb = (x.view(np.uint32) + np.uint32(0x7FFF) + ((x.view(np.uint32) >> 16) & 1) >> 16).astype(np.uint16)
            for l in range(L):
                sel = sel_of[(it, l)][t]
                ptrs = (C.c_void_p * len(sel))(*[expert(l, e).ctypes.data for e in sel])
                w = np.array([scores[it, l, t, e] for e in sel], dtype=np.float64)
                if renorm:
                    w = w / w.sum()
                wts = (w * rscale).astype(np.float32)
                xn = np.empty(d, dtype=np.uint16)
                cm.cpu_moe_layer(xb.ctypes.data, d, F, S, E, cache[("r", l)].ctypes.data,
                                 cache[("s", l)].ctypes.data if S else None,
                                 cache[("g", l)].ctypes.data if sg else None, ptrs, wts.ctypes.data, len(sel),
                                 logits.ctypes.data, y.ctypes.data, xn.ctypes.data, nthreads)
                xb = xn
    arith_s = time.perf_counter() - t0
    host_gbs = cm.cpu_bytes_touched() / arith_s / 1e9
    ms_token = arith_s * 1e3 / len(sample) + dec_ms_token  # per decode step (B tokens)
    kind = "reference" if use_ref else "port"
    sample_desc = (f"decisions: {'reference simulate() (oracle/_ref)' if use_ref else 'oracle C port'} over all "
                   f"{T} steps ({dec_ms_token:.3f} ms/step, 1 thread); arithmetic: oracle/cpu_moe.c fp32 over "
                   f"bf16 host weights, last {len(sample)} steps x {B} tokens x {L} layers "
                   f"({arith_s * 1e3 / len(sample):.1f} ms/step, {nthreads} threads, {host_gbs:.1f} GB/s of host "
                   f"weight reads)")
    return ms_token, kind, nthreads, sample_desc, host_gbs


def cpu_baseline(scores, x_host, n_tokens):
    nthreads = os.cpu_count() or 1
    ms, kind, cores, sample, gbs = cpu_path(scores, x_host, n_tokens, nthreads)
    return {"value": round(ms, 3), "unit": "ms/token", "cores": cores, "kind": kind, "sample": sample,
            "host_weight_gbs": round(gbs, 1)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    L, E, B, d = CFG["num_layers"], CFG["experts"], CFG["batch"], MODEL["d_model"]
    W, K = args.warmup, args.steps
    T = max(TOKENS, W + K)  # the same 512-token stream as the device arm
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import pyoracle as po
    scores = po.generate_trace(L, E, B, T, 7, use_ref=po.ref() is not None)
    x_host = ar1_hidden(T, B, d, 7)
    nthreads = os.cpu_count() or 1
    ms, kind, cores, sample, gbs = cpu_path(scores, x_host, min(args.cpu_sample_tokens, K), nthreads)
    print(json.dumps({
        "impl": "reference",
        "metric": "MoE decode ms/token + expert cache hit rate, DeepSeek-V2-Lite shape",
        "value": round(ms, 3), "unit": "ms/token", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": K, "warmup": W, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32 compute over bf16 weights; fp64 decisions", "data": "synthetic",
        "config": {"workload": f"DeepSeek-V2-Lite 26-layer MoE stack, batch-1 decode of a {T}-token stream "
                               f"(timed: its last {K} tokens), cache 16/64 experts per layer, CE+ER+Pre+BA "
                               "alpha=0.25", "stream_tokens": T},
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms/token", "cores": cores, "kind": kind, "sample": sample,
                         "host_weight_gbs": round(gbs, 1)},
        "e2e": {"value": round(ms, 3), "unit": "ms/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=TOKENS - 16)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-ablation", action="store_true")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batched", action="store_true", help="skip the batched (config C5) tensor-core FFN section")
    ap.add_argument("--cpu-sample-tokens", type=int, default=12)
    ap.add_argument("--no-c5", action="store_true", help="skip the stream-partitioned config C5 section")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
