// moe_stack_main.cpp — drives the C++ real-layer API (moesched::MoeStack,
// include/moesched/moe_layer.hpp) on the GPU the way a C++ caller of the
// reference library would, and prints the per-step decisions it gets back
// (RouteResult / load-list vocabulary) as JSON in the schema of the oracle's
// per-step records, plus the fp32 router scores the device used and the
// Metrics. tests/test_moe_stack_cpp.py replays the oracle on those scores and
// requires bit-exact equality.
//
//   moe_stack_main L E k B d F S slots T [er] [ba]
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "moesched/moe_layer.hpp"
#include "moesched_b200.h"

using namespace moesched;

static void list(const std::vector<std::uint32_t>& v) {
    std::printf("[");
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s%u", i ? "," : "", v[i]);
    std::printf("]");
}

int main(int argc, char** argv) {
    if (argc < 10) {
        std::fprintf(stderr, "usage: %s L E k B d F S slots T [er] [ba]\n", argv[0]);
        return 2;
    }
    auto u = [&](int i) { return (std::uint32_t)std::strtoul(argv[i], nullptr, 10); };
    const std::uint32_t L = u(1), E = u(2), k = u(3), B = u(4), d = u(5), F = u(6), S = u(7), slots = u(8), T = u(9);
    SimConfig cfg;
    cfg.shape = {L, E, k, B};
    cfg.router.alpha = 0.25;
    cfg.cache.slots_per_layer = slots;
    cfg.stages = StageSet::all();
    if (argc > 10) cfg.stages.er = u(10) != 0;
    if (argc > 11) cfg.stages.ba = u(11) != 0;
    cfg.seed = 7;
    ModelDims dims;
    dims.d_model = d;
    dims.ffn = F;
    dims.shared_ffn = S;
    dims.weight_seed = 7;
    try {
        MoeStack st(cfg, dims);
        // trace-driven routing: logits = ln(s) of the reference generator's scores
        std::vector<double> sc((size_t)T * L * B * E);
        if (moeb_generate_trace(L, E, B, 0.125, 0.8, 0.92, 1.5, T, 7, sc.data()) != 0) throw std::runtime_error(moeb_last_error());
        std::vector<float> lg(sc.size());
        for (size_t i = 0; i < sc.size(); ++i) lg[i] = sc[i] > 0 ? (float)std::log(sc[i]) : -INFINITY;  // capi.trace_logits
        st.set_logits_trace(lg.data(), T, T);
        void *x = nullptr, *y = nullptr;
        cudaMalloc(&x, (size_t)B * d * 2);
        cudaMalloc(&y, (size_t)B * d * 2);
        cudaMemset(x, 0x3c, (size_t)B * d * 2);  // bf16 ~1.0x
        for (std::uint32_t i = 0; i < T; ++i) st.step(x, y, B);
        st.sync();
        const std::vector<StepDecision> dec = st.decisions();
        const std::vector<float> scores = st.scores();
        const Metrics m = st.metrics();
        std::printf("{\"steps\":[");
        for (size_t i = 0; i < dec.size(); ++i) {
            const StepDecision& s = dec[i];
            std::vector<std::uint32_t> mask;
            for (std::uint32_t e = 0; e < E; ++e)
                if (s.resident_before[e]) mask.push_back(e);
            std::printf("%s{\"it\":%llu,\"layer\":%u,\"mask\":", i ? "," : "", (unsigned long long)s.iteration, s.layer);
            list(mask);
            std::printf(",\"tok\":[");
            for (size_t t = 0; t < s.route.tokens.size(); ++t) {
                const TokenRoute& tr = s.route.tokens[t];
                std::printf("%s{\"sel\":", t ? "," : "");
                list(tr.selected);
                std::printf(",\"sub\":[");
                for (size_t j = 0; j < tr.substitutions.size(); ++j)
                    std::printf("%s[%u,%u]", j ? "," : "", tr.substitutions[j].dropped, tr.substitutions[j].chosen);
                std::printf("],\"kept\":");
                list(tr.kept_low);
                std::printf("}");
            }
            std::printf("],\"load\":");
            list(s.load_list);
            std::printf(",\"cpu\":");
            list(s.cpu_list);
            std::printf(",\"pref\":");
            list(s.prefetched);
            std::printf(",\"evict\":[");
            for (size_t j = 0; j < s.evictions.size(); ++j)
                std::printf("%s[%u,%u]", j ? "," : "", s.evictions[j].layer, s.evictions[j].expert);
            std::printf("],\"completion\":%llu,\"pending\":", (unsigned long long)s.completion);
            list(s.route.pending);
            std::printf("}");
        }
        std::printf("],\"scores\":[");
        for (size_t i = 0; i < scores.size(); ++i) std::printf("%s%.9g", i ? "," : "", scores[i]);
        std::printf("],\"metrics\":{\"hits\":%llu,\"misses\":%llu,\"selections\":%llu,\"demand_loads\":%llu,"
                    "\"cpu_computed\":%llu,\"prefetch_loads\":%llu,\"substitutions\":%llu,\"low_score_kept\":%llu,"
                    "\"iterations\":%llu,\"total_time\":%llu,\"stage\":\"%s\"}}\n",
                    (unsigned long long)m.hits, (unsigned long long)m.misses, (unsigned long long)m.selections,
                    (unsigned long long)m.demand_loads, (unsigned long long)m.cpu_computed,
                    (unsigned long long)m.prefetch_loads, (unsigned long long)m.substitutions,
                    (unsigned long long)m.low_score_kept, (unsigned long long)m.iterations,
                    (unsigned long long)m.total_time, m.stage.c_str());
        cudaFree(x);
        cudaFree(y);
        // prefill of a 40-token prompt: the uploads of the non-resident
        // experts, bitwise-reproducible hidden outputs, decisions unchanged
        if (F % 128 == 0 && S % 128 == 0) {
            const std::uint32_t N = 40;
            void *px = nullptr, *py0 = nullptr, *py1 = nullptr;
            cudaMalloc(&px, (size_t)N * d * 2);
            cudaMalloc(&py0, (size_t)N * d * 2);
            cudaMalloc(&py1, (size_t)N * d * 2);
            std::vector<std::uint16_t> hx((size_t)N * d);
            for (size_t i = 0; i < hx.size(); ++i) hx[i] = (std::uint16_t)(0x3c00u + (i * 2654435761u >> 20) % 512u);
            cudaMemcpy(px, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
            const std::uint64_t up = st.prefill(px, py0, N);
            st.prefill(px, py1, N);
            st.sync();
            std::vector<std::uint16_t> a(hx.size()), b(hx.size());
            cudaMemcpy(a.data(), py0, a.size() * 2, cudaMemcpyDeviceToHost);
            cudaMemcpy(b.data(), py1, b.size() * 2, cudaMemcpyDeviceToHost);
            const bool same = a == b, decisions_kept = st.decisions().size() == dec.size();
            std::fprintf(stderr, "prefill h2d %llu reproducible %d decisions_kept %d\n", (unsigned long long)up,
                         (int)same, (int)decisions_kept);
            cudaFree(px);
            cudaFree(py0);
            cudaFree(py1);
            const std::uint64_t want = (std::uint64_t)L * (E - std::min(slots, E)) * 3ull * F * d * 2;
            if (up != want || !same || !decisions_kept) {
                std::fprintf(stderr, "prefill check failed (want %llu)\n", (unsigned long long)want);
                return 1;
            }
        }
        // the reference's exception types come back through the wrapper
        try {
            SimConfig bad = cfg;
            bad.shape.batch_size = 64;
            MoeStack oops(bad, dims);
            std::fprintf(stderr, "expected ConfigError\n");
            return 1;
        } catch (const ConfigError&) {
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
