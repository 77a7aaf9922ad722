"""Per-CTA phase stamps of the batch-1 split-K FFN inside the pipeline
(MOEB_FFN_TSTAMP=1, moeb_debug_ffn_tstamps): DSV2-Lite 26 layers, the last
layer's FFN of each of the last K tokens. Prints, relative to the earliest
CTA entry, the median over tokens of the min / median / max over CTAs of
each phase stamp.

  python tools/ffn_phases.py [--allhit] [--tokens 24]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

os.environ["MOEB_FFN_TSTAMP"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

NAMES = ["entry", "shared issued", "certain released", "certain issued", "final plan in hand", "all rows issued",
         "consumers done", "end"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--allhit", action="store_true")
    ap.add_argument("--tokens", type=int, default=24)
    args = ap.parse_args()
    import torch
    from paper_2508_18983_b200 import capi
    L, E, B, d, T = 26, 64, 1, 2048, args.tokens
    cfg = capi.Config.make(num_layers=L, experts=E, top_k=6, batch=B, slots=E if args.allhit else 16)
    st = capi.Stack(cfg, 2048, 1408, 2816, weight_seed=7)
    st.set_logits_trace(capi.trace_logits(capi.generate_trace(L, E, B, T, 7)), T)
    x = torch.randn(T, B, d).to(torch.bfloat16).cuda()
    y = torch.empty(B, d, dtype=torch.bfloat16, device="cuda")
    lib = capi.lib()
    rows = []
    for i in range(T):
        st.step(x[i].data_ptr(), y.data_ptr(), B)
        st.sync()
        n = C.c_size_t(0)
        buf = np.zeros(8 * 256, dtype=np.uint64)  # >= 8 words per SM
        capi.check(lib.moeb_debug_ffn_tstamps(st.h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), C.c_size_t(buf.size),
                                              C.byref(n)))
        if i >= T // 3:
            rows.append(buf.reshape(-1, 8).astype(np.int64).copy())
    st.close()
    stats = []
    for r in rows:
        r = r[r[:, 0] != 0]
        t0 = r[:, 0].min()
        per = []
        for j in range(8):
            v = r[:, j]
            v = v[v != 0]
            per.append((np.min(v) - t0, np.median(v) - t0, np.max(v) - t0) if len(v) else (np.nan,) * 3)
        stats.append(per)
    stats = np.array(stats, dtype=np.float64) / 1e3
    med = np.nanmedian(stats, axis=0)
    print(f"{'phase':22s} {'min':>8s} {'median':>8s} {'max':>8s}  (us after the first CTA entry; median over "
          f"{len(rows)} tokens, layer {L - 1}, {'all-resident' if args.allhit else 'cache 16/64'})")
    for j, nm in enumerate(NAMES):
        print(f"{nm:22s} {med[j, 0]:8.2f} {med[j, 1]:8.2f} {med[j, 2]:8.2f}")


if __name__ == "__main__":
    main()
