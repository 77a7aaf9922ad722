// moe_stack.cpp — moesched::MoeStack (include/moesched/moe_layer.hpp) over
// the C-ABI: decisions come back as plain records (moeb_get_decisions) and are
// turned into the reference's RouteResult / Metrics vocabulary
// (router.hpp:38-54, pipeline.hpp:63-78).
#include <algorithm>
#include <stdexcept>
#include <utility>

#include "moesched/moe_layer.hpp"
#include "moesched_b200.h"

namespace moesched {

void throw_status(int rc);                    // policies.cpp
moeb_config to_moeb_config(const SimConfig&);  // sim.cpp

MoeStack::MoeStack(const SimConfig& cfg, const ModelDims& dims, const void* host_pool, int device,
                   bool record_decisions)
    : cfg_(cfg), dims_(dims) {
    const moeb_config c = to_moeb_config(cfg);
    moeb_model m{};
    m.d_model = dims.d_model;
    m.ffn = dims.ffn;
    m.shared_ffn = dims.shared_ffn;
    m.shared_gate = dims.shared_gate ? 1 : 0;
    m.renormalize = dims.renormalize ? 1 : 0;
    m.routed_scale = dims.routed_scale;
    m.weight_seed = dims.weight_seed;
    m.max_batch = cfg.shape.batch_size;
    m.flags = record_decisions ? MOEB_MODEL_LOG_STEPS : 0u;
    throw_status(moeb_create(&c, &m, host_pool, device, &h_));
}

MoeStack::~MoeStack() {
    if (h_) moeb_destroy(h_);
}

MoeStack::MoeStack(MoeStack&& o) noexcept : cfg_(o.cfg_), dims_(o.dims_), h_(std::exchange(o.h_, nullptr)) {}

MoeStack& MoeStack::operator=(MoeStack&& o) noexcept {
    if (this != &o) {
        if (h_) moeb_destroy(h_);
        cfg_ = o.cfg_;
        dims_ = o.dims_;
        h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
}

void MoeStack::set_logits_trace(const float* logits, std::uint64_t n_steps, std::uint64_t total_iterations) {
    throw_status(moeb_set_logits_trace(h_, logits, n_steps, total_iterations));
}

void MoeStack::step(const void* x, void* y, std::uint32_t batch, void* stream) {
    throw_status(moeb_step(h_, x, y, batch, stream));
}

void MoeStack::sync() { throw_status(moeb_sync(h_)); }

std::uint64_t MoeStack::prefill(const void* x, void* y, std::uint32_t n_tokens, void* stream) {
    std::uint64_t bytes = 0;
    throw_status(moeb_prefill(h_, x, y, n_tokens, stream, &bytes));
    return bytes;
}

void MoeStack::reset() { throw_status(moeb_reset(h_)); }

Metrics MoeStack::metrics() const {
    moeb_metrics m{};
    throw_status(moeb_get_metrics(h_, &m));
    Metrics out;
    out.stage = cfg_.stages.label();
    out.tpot = m.tpot;
    out.hit_rate = m.hit_rate;
    out.substitution_ratio = m.substitution_ratio;
    out.demand_loads = m.demand_loads;
    out.prefetch_loads = m.prefetch_loads;
    out.cpu_computed = m.cpu_computed;
    out.hits = m.hits;
    out.misses = m.misses;
    out.substitutions = m.substitutions;
    out.low_score_kept = m.low_score_kept;
    out.selections = m.selections;
    out.iterations = m.iterations;
    out.total_time = m.total_time;
    return out;
}

std::vector<StepDecision> MoeStack::decisions() const {
    size_t n = 0;
    throw_status(moeb_get_decisions(h_, nullptr, nullptr, 0, &n));
    const std::uint32_t B = cfg_.shape.batch_size, E = cfg_.shape.experts_per_layer;
    std::vector<moeb_step_record> rs(n);
    std::vector<moeb_token_record> ts(n * B);
    throw_status(moeb_get_decisions(h_, rs.data(), ts.data(), n, &n));
    std::vector<StepDecision> out;
    out.reserve(n);
    for (size_t i = 0; i < n; ++i) {
        const moeb_step_record& r = rs[i];
        StepDecision d;
        d.iteration = r.iteration;
        d.layer = r.layer;
        d.completion = r.completion;
        d.resident_before.assign(E, 0);
        for (std::uint32_t e = 0; e < E; ++e) d.resident_before[e] = (r.resident_before >> e) & 1u;
        std::vector<std::uint32_t> pending;
        for (std::uint32_t t = 0; t < B; ++t) {
            const moeb_token_record& tr = ts[i * B + t];
            TokenRoute tok;
            tok.selected.assign(tr.sel, tr.sel + tr.n_sel);
            for (std::uint32_t s = 0; s < tr.n_sub; ++s) tok.substitutions.push_back({tr.sub_dropped[s], tr.sub_chosen[s]});
            tok.kept_low.assign(tr.kept, tr.kept + tr.n_kept);
            pending.insert(pending.end(), tok.kept_low.begin(), tok.kept_low.end());
            d.route.tokens.push_back(std::move(tok));
        }
        // pending = the kept low-score experts not resident (router.cpp:150), sorted unique
        std::sort(pending.begin(), pending.end());
        pending.erase(std::unique(pending.begin(), pending.end()), pending.end());
        for (std::uint32_t e : pending)
            if (!d.resident_before[e]) d.route.pending.push_back(e);
        d.load_list.assign(r.load, r.load + r.n_load);
        d.cpu_list.assign(r.cpu, r.cpu + r.n_cpu);
        d.prefetched.assign(r.pref, r.pref + r.n_pref);
        for (std::uint32_t s = 0; s < r.n_evict; ++s)
            d.evictions.push_back({r.completion, r.evict_layer[s], r.evict_expert[s]});
        out.push_back(std::move(d));
    }
    return out;
}

std::vector<float> MoeStack::scores() const {
    size_t n = 0;
    throw_status(moeb_get_scores(h_, nullptr, 0, &n));
    std::vector<float> v(n);
    throw_status(moeb_get_scores(h_, v.data(), n, &n));
    return v;
}

std::vector<float> MoeStack::layer_outputs() const {
    std::vector<float> v((size_t)cfg_.shape.num_layers * cfg_.shape.batch_size * dims_.d_model);
    throw_status(moeb_get_layer_outputs(h_, v.data(), v.size()));
    return v;
}

}  // namespace moesched
