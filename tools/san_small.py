"""A small stack (B = 1 split-K and B = 2 tcgen05 FFN) for compute-sanitizer runs
(tools/gpu_sanitize.sh): the stack detects the tool and runs in serial mode.
Each stack also runs a prefill of 150 tokens (re-tiled for B = 1)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2508_18983_b200 import capi
for B, F, S in ((1, 128, 256), (2, 128, 256)):
    kw = dict(num_layers=2, experts=16, top_k=4, batch=B, slots=4, alpha=0.25, seed=7)
    st = capi.Stack(capi.Config.make(**kw), 256, F, S, weight_seed=7, log_steps=True)
    st.set_logits_trace(capi.trace_logits(capi.generate_trace(2, 16, B, 6, 7)), 6)
    x = torch.randn(6, B, 256).to(torch.bfloat16).cuda()
    y = torch.empty(B, 256, dtype=torch.bfloat16, device="cuda")
    for i in range(6):
        st.step(x[i].data_ptr(), y.data_ptr(), B)
    st.sync()
    xp = torch.randn(150, 256).to(torch.bfloat16).cuda()
    yp = torch.empty_like(xp)
    up = st.prefill(xp.data_ptr(), yp.data_ptr(), 150)
    st.sync()
    print("B", B, "ok", st.metrics()["hits"], "prefill uploaded", up)
    st.close()
