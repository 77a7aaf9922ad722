"""Prefill (moeb_prefill) throughput on one B200: DeepSeek-V2-Lite, 26 layers,
a prompt of N tokens, time to first token (TTFT, all layers) with

  * every expert resident in HBM (cache 64/64): HBM / tensor-core bound;
  * the capped cache (16/64): the paper's prefill pipeline, the 48 other
    experts of each layer uploaded from the pinned pool while the previous
    layer computes — PCIe-bound.

Roofline per prompt: T_roof = sum over layers of max(weight bytes / HBM
peak, FLOPs / bf16 tensor peak) (MEASURED_PEAKS.json), and for the capped
cache max(that, upload bytes / the measured PCIe rate). The CPU baseline is
oracle/cpu_moe.c's batched prefill layer (cpu_moe_prefill_layer) on every
host thread, one layer timed and scaled by L.

  python tools/bench_prefill.py [--tokens 128,512,2048,4096] [--out f.json]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

L, E, K, D, F, S = 26, 64, 6, 2048, 1408, 2816


def peaks():
    with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
        p = json.load(f)
    return p["hbm_gbs"], p["bf16_tflops"]


def pcie_gbs(torch):
    h = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
    g = torch.empty_like(h, device="cuda")
    g.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):  # the best of three 1 GiB trials
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            g.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, 4 * h.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def time_prefill(torch, st, x, y, N, reps):
    s = torch.cuda.Stream()  # a real stream handle (0 would select the stack's own stream)
    st.prefill(x.data_ptr(), y.data_ptr(), N, stream=s.cuda_stream)  # warm-up (buffers, first launches)
    st.prefill(x.data_ptr(), y.data_ptr(), N, stream=s.cuda_stream)
    torch.cuda.synchronize()
    ts, up = [], 0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        up = st.prefill(x.data_ptr(), y.data_ptr(), N, stream=s.cuda_stream)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), up


def roofline(N, n_used, hbm, tflops):
    """Per prompt: weights of the shared + used experts (+ router), FLOPs of
    every (token, expert) pair; the activation traffic is listed beside."""
    wbytes = L * (E * D * 2 + 3 * S * D * 2) + n_used * 3 * F * D * 2
    flops = L * 2 * 3 * D * (N * S + N * K * F)
    t_hbm, t_tc = wbytes / (hbm * 1e9) * 1e3, flops / (tflops * 1e12) * 1e3
    return wbytes, flops, t_hbm, t_tc


def cpu_prefill_ms(N, nthreads):
    """One DSV2-Lite layer of cpu_moe_prefill_layer at N tokens, x L."""
    cm = C.CDLL(os.path.join(REPO, "oracle", "libcpumoe.so"))
    cm.cpu_synth.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p, C.c_int]
    cm.cpu_moe_prefill_layer.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                         C.c_float, C.c_void_p, C.c_void_p, C.c_int]
    cm.cpu_bytes_touched.restype = C.c_uint64
    l = 3

    def synth(tid, n, fan_in):
        a = np.empty(n, dtype=np.uint16)
        cm.cpu_synth(7, tid, n, fan_in, a.ctypes.data, nthreads)
        return a

    router = synth((l << 20) | (0xFFFF << 4), E * D, D)
    shared = np.concatenate([synth((l << 20) | (0xFFFE << 4) | m, S * D, D if m < 2 else S) for m in range(3)])
    experts = [np.concatenate([synth((l << 20) | (e << 4) | m, F * D, D if m < 2 else F) for m in range(3)])
               for e in range(E)]
    ptrs = (C.c_void_p * E)(*[a.ctypes.data for a in experts])
    rng = np.random.default_rng(1)
    xf = (rng.standard_normal((N, D)) * 2).astype(np.float32)
    x = ((xf.view(np.uint32) + np.uint32(0x7FFF) + ((xf.view(np.uint32) >> 16) & 1)) >> 16).astype(np.uint16)
    xn = np.empty_like(x)
    cm.cpu_bytes_touched()
    t0 = time.perf_counter()
    cm.cpu_moe_prefill_layer(x.ctypes.data, N, D, F, S, E, K, router.ctypes.data, shared.ctypes.data, None, ptrs, 0,
                             1.0, xn.ctypes.data, None, nthreads)
    dt = time.perf_counter() - t0
    return dt * 1e3 * L, cm.cpu_bytes_touched() / dt / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="128,512,2048,4096")
    ap.add_argument("--capped-tokens", default="512")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu-tokens", type=int, default=512)
    ap.add_argument("--rows", type=int, default=512, help="also time a batch-1 (row-interleaved, re-tiled) "
                    "capped stack at this N (0: skip)")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    from paper_2508_18983_b200 import partition
    partition.bind_to_device_node(0)  # pinned pools first-touched on the GPU's NUMA node
    import torch
    from paper_2508_18983_b200 import capi
    hbm, tflops = peaks()
    bw_pcie = pcie_gbs(torch)
    out = {"workload": f"DeepSeek-V2-Lite {L} layers, one prompt of N tokens, plain top-{K} routing, grouped tcgen05 "
                       "GEMM; TTFT = all layers, CUDA events on the stream", "hbm_peak_gbs": hbm,
           "bf16_peak_tflops": tflops, "pcie_gbs": round(bw_pcie, 2), "resident": {}, "capped": {}}
    t0 = time.time()
    model = dict(d_model=D, ffn=F, shared_ffn=S, shared_gate=0, renormalize=0, routed_scale=1.0)
    capped = capi.Stack(capi.Config.make(num_layers=L, experts=E, top_k=K, batch=2, slots=16), weight_seed=7,
                        log_steps=False, **model)
    full = capi.Stack(capi.Config.make(num_layers=L, experts=E, top_k=K, batch=2, slots=64), weight_seed=7,
                      weights_host=(capped.host_pool()[0], capped), **model)
    out["create_s"] = round(time.time() - t0, 1)
    toks = [int(t) for t in args.tokens.split(",") if t]
    nmax = max(toks + [int(t) for t in args.capped_tokens.split(",") if t])
    g = torch.Generator().manual_seed(7)
    xall = (torch.randn(nmax, D, generator=g) * 2).to(torch.bfloat16).cuda()
    y = torch.empty_like(xall)
    for N in toks:
        ms, _ = time_prefill(torch, full, xall[:N], y[:N], N, args.reps)
        # every expert is used by a prompt of >= 128 tokens (p(unused) < 1e-5)
        wb, fl, t_hbm, t_tc = roofline(N, L * E, hbm, tflops)
        t_roof = max(t_hbm, t_tc)
        out["resident"][f"N{N}"] = {
            "ttft_ms": round(ms, 3), "tokens_per_s": round(N / (ms * 1e-3), 1),
            "weight_gb": round(wb / 1e9, 3), "tflop": round(fl / 1e12, 3),
            "achieved_gbs": round(wb / (ms * 1e-3) / 1e9, 1), "achieved_tflops": round(fl / (ms * 1e-3) / 1e12, 1),
            "roofline": {"t_roof_ms": round(t_roof, 3), "bound": "hbm" if t_hbm >= t_tc else "tensor",
                         "frac": round(t_roof / ms, 4)}}
        print(json.dumps({f"resident N{N}": out["resident"][f"N{N}"]}), flush=True)
    for N in [int(t) for t in args.capped_tokens.split(",") if t]:
        ms, up = time_prefill(torch, capped, xall[:N], y[:N], N, max(2, args.reps // 2))
        wb, fl, t_hbm, t_tc = roofline(N, L * E, hbm, tflops)
        t_pcie = up / (bw_pcie * 1e9) * 1e3
        t_roof = max(t_hbm, t_tc, t_pcie)
        out["capped"][f"N{N}"] = {
            "ttft_ms": round(ms, 3), "tokens_per_s": round(N / (ms * 1e-3), 1), "upload_gb": round(up / 1e9, 3),
            "pcie_achieved_gbs": round(up / (ms * 1e-3) / 1e9, 2),
            "roofline": {"t_roof_ms": round(t_roof, 3), "bound": "pcie" if t_pcie >= max(t_hbm, t_tc) else "hbm",
                         "frac": round(t_roof / ms, 4)}}
        print(json.dumps({f"capped N{N}": out["capped"][f"N{N}"]}), flush=True)
    full.close()
    capped.close()
    if args.rows:
        # the headline decode stack (batch 1: split-K layout), prefill through the re-tiling pass
        N = args.rows
        rows = capi.Stack(capi.Config.make(num_layers=L, experts=E, top_k=K, batch=1, slots=16), weight_seed=7,
                          **model)
        ms, up = time_prefill(torch, rows, xall[:N], y[:N], N, 2)
        wb, fl, t_hbm, t_tc = roofline(N, L * E, hbm, tflops)
        t_pcie = up / (bw_pcie * 1e9) * 1e3
        t_roof = max(t_hbm, t_tc, t_pcie)
        out["capped_batch1_stack"] = {
            "N": N, "ttft_ms": round(ms, 3), "tokens_per_s": round(N / (ms * 1e-3), 1), "upload_gb": round(up / 1e9, 3),
            "roofline": {"t_roof_ms": round(t_roof, 3), "bound": "pcie" if t_pcie >= max(t_hbm, t_tc) else "hbm",
                         "frac": round(t_roof / ms, 4)}}
        print(json.dumps({"capped_batch1_stack": out["capped_batch1_stack"]}), flush=True)
        rows.close()
    if args.cpu_tokens:
        nthreads = os.cpu_count() or 1
        ms, gbs = cpu_prefill_ms(args.cpu_tokens, nthreads)
        out["cpu_baseline"] = {"value": round(ms, 1), "unit": "ms TTFT", "tokens": args.cpu_tokens, "cores": nthreads,
                               "kind": "port", "sample": f"oracle/cpu_moe.c cpu_moe_prefill_layer (batched per expert, "
                               f"AVX2 fp32 over bf16 host weights), one layer at N={args.cpu_tokens} timed x {L} "
                               f"layers, {nthreads} threads, {gbs:.1f} GB/s of weight reads"}
        print(json.dumps({"cpu_baseline": out["cpu_baseline"]}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
