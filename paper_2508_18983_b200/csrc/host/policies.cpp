// policies.cpp — router / cache / prefetch / balancer members of the moesched
// drop-in API, executed on the B200 through the C-ABI (include/moesched_b200.h).
// Reference behaviour: /root/reference/proj/src/{router,cache,prefetch,balancer}.cpp.
#include <algorithm>
#include <stdexcept>
#include <string>

#include "moesched/balancer.hpp"
#include "moesched/cache.hpp"
#include "moesched/prefetch.hpp"
#include "moesched/router.hpp"
#include "moesched_b200.h"

namespace moesched {

// Status code of the C-ABI -> the reference's exception type and message.
void throw_status(int rc) {
    if (rc == MOEB_OK) return;
    const std::string msg = moeb_last_error();
    switch (rc) {
        case MOEB_ECONFIG: throw ConfigError(msg);
        case MOEB_EIO: throw IoError(msg);
        case MOEB_ECACHE: throw CacheError(msg);
        case MOEB_ELOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error("CUDA: " + msg);
    }
}

namespace {

std::vector<double> flatten(const std::vector<std::vector<double>>& rows, std::uint32_t& E) {
    E = rows.empty() ? 0 : static_cast<std::uint32_t>(rows[0].size());
    std::vector<double> flat;
    flat.reserve(rows.size() * E);
    for (const auto& r : rows) flat.insert(flat.end(), r.begin(), r.end());
    return flat;
}

std::vector<std::uint32_t> sorted_unique(std::vector<std::uint32_t> v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    return v;
}

}  // namespace

// -------------------------------------------------------------------- router
Classification classify(std::span<const double> scores, std::uint32_t k, double alpha) {
    const std::uint32_t E = static_cast<std::uint32_t>(scores.size());
    if (E <= k) throw ConfigError("classify: beta undefined, need at least k+1 experts");
    double thr[4];
    std::vector<std::uint32_t> act(E), top(E), low(E), alt(E);
    std::uint32_t nt = 0, nl = 0, na = 0;
    throw_status(moeb_classify(scores.data(), E, k, alpha, thr, act.data(), top.data(), &nt, low.data(), &nl,
                               alt.data(), &na));
    Classification c;
    c.beta = thr[0];
    c.threshold_top = thr[1];
    c.threshold_low = thr[2];
    c.threshold_alt = thr[3];
    c.actives.assign(act.begin(), act.begin() + k);
    c.top_score.assign(top.begin(), top.begin() + nt);
    c.low_score.assign(low.begin(), low.begin() + nl);
    c.alt_band.assign(alt.begin(), alt.begin() + na);
    return c;
}

std::vector<std::uint32_t> RouteResult::distinct_selected() const {
    std::vector<std::uint32_t> all;
    for (const TokenRoute& t : tokens) all.insert(all.end(), t.selected.begin(), t.selected.end());
    return sorted_unique(std::move(all));
}

std::uint64_t RouteResult::substitution_count() const {
    std::uint64_t n = 0;
    for (const TokenRoute& t : tokens) n += t.substitutions.size();
    return n;
}

std::uint64_t RouteResult::kept_low_count() const {
    std::uint64_t n = 0;
    for (const TokenRoute& t : tokens) n += t.kept_low.size();
    return n;
}

namespace {

struct RouteBuffers {
    std::vector<std::uint32_t> sel, nsel, sub, nsub, kept, nkept, cset, pend;
    std::uint32_t nc = 0, np = 0;
    RouteBuffers(std::uint32_t B, std::uint32_t E, std::uint32_t k)
        : sel(B * k), nsel(B), sub(2 * B * k), nsub(B), kept(B * k), nkept(B), cset(E), pend(E) {}
};

void unpack(RouteResult& r, const RouteBuffers& b, std::uint32_t B, std::uint32_t k, bool with_c) {
    for (std::uint32_t t = 0; t < B; ++t) {
        TokenRoute& tk = r.tokens[t];
        tk.selected.assign(b.sel.begin() + t * k, b.sel.begin() + t * k + b.nsel[t]);
        tk.kept_low.assign(b.kept.begin() + t * k, b.kept.begin() + t * k + b.nkept[t]);
        tk.substitutions.clear();
        for (std::uint32_t i = 0; i < b.nsub[t]; ++i)
            tk.substitutions.push_back({b.sub[(t * k + i) * 2], b.sub[(t * k + i) * 2 + 1]});
    }
    if (with_c) r.top_score_set.assign(b.cset.begin(), b.cset.begin() + b.nc);
    r.pending.assign(b.pend.begin(), b.pend.begin() + b.np);
}

}  // namespace

RouteResult route(const std::vector<std::vector<double>>& batch_scores, std::span<const std::uint8_t> resident_mask,
                  std::uint32_t k, double alpha) {
    RouteResult r;
    const std::uint32_t B = static_cast<std::uint32_t>(batch_scores.size());
    r.tokens.resize(B);
    if (B == 0) return r;
    std::uint32_t E = 0;
    const std::vector<double> flat = flatten(batch_scores, E);
    if (E <= k) throw ConfigError("classify: beta undefined, need at least k+1 experts");
    RouteBuffers b(B, E, k);
    throw_status(moeb_route(flat.data(), B, E, resident_mask.data(), k, alpha, 0, b.sel.data(), b.nsel.data(),
                            b.sub.data(), b.nsub.data(), b.kept.data(), b.nkept.data(), b.cset.data(), &b.nc,
                            b.pend.data(), &b.np));
    unpack(r, b, B, k, true);
    for (std::uint32_t t = 0; t < B; ++t) r.tokens[t].cls = classify(batch_scores[t], k, alpha);
    return r;
}

RouteResult coalesce_for_batching(const RouteResult& result, const std::vector<std::vector<double>>& batch_scores,
                                  std::span<const std::uint8_t> resident_mask) {
    RouteResult out = result;
    const std::uint32_t B = static_cast<std::uint32_t>(out.tokens.size());
    if (B == 0) return out;
    std::uint32_t E = 0;
    const std::vector<double> flat = flatten(batch_scores, E);
    std::uint32_t k = 0;
    for (const TokenRoute& t : out.tokens) k = std::max<std::uint32_t>(k, static_cast<std::uint32_t>(t.selected.size()));
    RouteBuffers b(B, E, std::max<std::uint32_t>(k, 1));
    const std::uint32_t kk = std::max<std::uint32_t>(k, 1);
    for (std::uint32_t t = 0; t < B; ++t) {
        const TokenRoute& tk = out.tokens[t];
        b.nsel[t] = static_cast<std::uint32_t>(tk.selected.size());
        b.nkept[t] = static_cast<std::uint32_t>(tk.kept_low.size());
        b.nsub[t] = static_cast<std::uint32_t>(tk.substitutions.size());
        for (std::uint32_t i = 0; i < b.nsel[t]; ++i) b.sel[t * kk + i] = tk.selected[i];
        for (std::uint32_t i = 0; i < b.nkept[t]; ++i) b.kept[t * kk + i] = tk.kept_low[i];
        for (std::uint32_t i = 0; i < b.nsub[t]; ++i) {
            b.sub[(t * kk + i) * 2] = tk.substitutions[i].dropped;
            b.sub[(t * kk + i) * 2 + 1] = tk.substitutions[i].chosen;
        }
    }
    std::vector<double> thr(4 * B);
    for (std::uint32_t t = 0; t < B; ++t) {
        const Classification& c = out.tokens[t].cls;
        thr[4 * t] = c.beta;
        thr[4 * t + 1] = c.threshold_top;
        thr[4 * t + 2] = c.threshold_low;
        thr[4 * t + 3] = c.threshold_alt;
    }
    throw_status(moeb_coalesce(flat.data(), B, E, resident_mask.data(), kk, thr.data(), b.sel.data(), b.nsel.data(),
                               b.sub.data(), b.nsub.data(), b.kept.data(), b.nkept.data(),
                               out.top_score_set.data(), static_cast<std::uint32_t>(out.top_score_set.size()),
                               b.pend.data(), &b.np));
    unpack(out, b, B, kk, false);
    return out;
}

std::vector<std::uint32_t> plain_top_k(std::span<const double> scores, std::uint32_t k) {
    std::vector<std::uint32_t> out(std::max<size_t>(scores.size(), 1));
    std::uint32_t n = 0;
    throw_status(moeb_plain_top_k(scores.data(), static_cast<std::uint32_t>(scores.size()), k, out.data(), &n));
    out.resize(n);
    return out;
}

// --------------------------------------------------------------------- cache
CacheState::CacheState(const ModelShape& shape, const CacheConfig& cfg, std::uint64_t seed)
    : shape_(shape), cfg_(cfg) {
    throw_status(moeb_cache_create(shape.num_layers, shape.experts_per_layer, cfg.slots_per_layer,
                                   cfg.history_window, cfg.policy == CachePolicy::LRU ? 1 : 0,
                                   cfg.init_fill == InitFill::FirstSlots     ? 0
                                   : cfg.init_fill == InitFill::SeededRandom ? 1
                                                                             : 2,
                                   seed, &dev_));
    mirror_.resize(shape.num_layers);
    for (std::uint32_t l = 0; l < shape.num_layers; ++l) refresh(l);
}

CacheState::CacheState(CacheState&& o) noexcept
    : shape_(o.shape_), cfg_(o.cfg_), dev_(o.dev_), mirror_(std::move(o.mirror_)) {
    o.dev_ = nullptr;
}

CacheState& CacheState::operator=(CacheState&& o) noexcept {
    if (this != &o) {
        if (dev_) moeb_cache_destroy(dev_);
        shape_ = o.shape_;
        cfg_ = o.cfg_;
        dev_ = o.dev_;
        mirror_ = std::move(o.mirror_);
        o.dev_ = nullptr;
    }
    return *this;
}

CacheState::~CacheState() {
    if (dev_) moeb_cache_destroy(dev_);
}

void CacheState::refresh(std::uint32_t layer) const {
    Mirror& m = mirror_.at(layer);
    std::vector<std::uint32_t> res(shape_.experts_per_layer + 1);
    std::uint32_t n = 0;
    throw_status(moeb_cache_resident(dev_, layer, res.data(), &n));
    res.resize(n);
    m.resident = std::move(res);
    m.mask.assign(shape_.experts_per_layer, 0);
    for (std::uint32_t e : m.resident) m.mask[e] = 1;
}

const std::vector<std::uint32_t>& CacheState::resident(std::uint32_t layer) const { return mirror_.at(layer).resident; }

std::span<const std::uint8_t> CacheState::resident_mask(std::uint32_t layer) const { return mirror_.at(layer).mask; }

bool CacheState::is_resident(std::uint32_t layer, std::uint32_t index) const { return mirror_.at(layer).mask[index] != 0; }

void CacheState::record_scores(std::uint32_t layer, std::span<const double> scores) {
    mirror_.at(layer);
    throw_status(moeb_cache_record(dev_, layer, scores.data(), static_cast<std::uint32_t>(scores.size())));
}

double CacheState::window_average(std::uint32_t layer, std::uint32_t index) const {
    mirror_.at(layer);
    double v = 0.0;
    throw_status(moeb_cache_window_average(dev_, layer, index, &v));
    return v;
}

std::optional<std::uint32_t> CacheState::try_evict_candidate(std::uint32_t layer) const {
    mirror_.at(layer);
    std::int64_t v = -1;
    throw_status(moeb_cache_try_evict(dev_, layer, &v));
    if (v < 0) return std::nullopt;
    return static_cast<std::uint32_t>(v);
}

std::uint32_t CacheState::evict_candidate(std::uint32_t layer) const {
    const auto v = try_evict_candidate(layer);
    if (!v) throw CacheError("no evictable expert");
    return *v;
}

void CacheState::shield(std::uint32_t layer, std::uint32_t index) {
    mirror_.at(layer);
    throw_status(moeb_cache_shield(dev_, layer, index));
}

void CacheState::unshield_layer(std::uint32_t layer) {
    mirror_.at(layer);
    throw_status(moeb_cache_unshield_layer(dev_, layer));
}

bool CacheState::is_shielded(std::uint32_t layer, std::uint32_t index) const {
    mirror_.at(layer);
    std::int32_t v = 0;
    throw_status(moeb_cache_is_shielded(dev_, layer, index, &v));
    return v != 0;
}

void CacheState::touch(std::uint32_t layer, std::uint32_t index, TimeUnits now) {
    mirror_.at(layer);
    throw_status(moeb_cache_touch(dev_, layer, index, now));
}

std::optional<std::uint32_t> CacheState::admit(std::uint32_t layer, std::uint32_t index, TimeUnits now) {
    mirror_.at(layer);
    std::int64_t ev = -1;
    const int rc = moeb_cache_admit(dev_, layer, index, now, &ev);
    if (rc == MOEB_ELOGIC) throw std::logic_error("admit: expert already resident");
    throw_status(rc);
    refresh(layer);
    if (ev < 0) return std::nullopt;
    return static_cast<std::uint32_t>(ev);
}

std::vector<std::vector<std::uint32_t>> CacheState::snapshot() const {
    std::vector<std::vector<std::uint32_t>> out;
    for (const Mirror& m : mirror_) out.push_back(m.resident);
    return out;
}

// ------------------------------------------------------------------ prefetch
PredictOutcome predict_scores(std::span<const double> true_next, std::span<const double> supplied,
                              const PredictorConfig& cfg, std::uint32_t k, double alpha, Rng& rng) {
    PredictOutcome o;
    o.scores.resize(true_next.size());
    std::uint32_t head = 0;
    std::int32_t kind = 0;
    throw_status(moeb_predict_scores(true_next.data(), supplied.empty() ? nullptr : supplied.data(),
                                     static_cast<std::uint32_t>(true_next.size()), cfg.p_top, cfg.p_active, k,
                                     alpha, rng.raw_state(), o.scores.data(), &head, &kind));
    o.head = head;
    o.head_kind = static_cast<PredictedHeadKind>(kind);
    o.from_trace = !supplied.empty();
    return o;
}

PrefetchQueue build_queue(std::span<const double> predicted, std::span<const std::uint8_t> resident_mask,
                          std::uint32_t depth, std::uint32_t target_layer, std::uint64_t target_iteration) {
    PrefetchQueue q;
    q.target_layer = target_layer;
    q.target_iteration = target_iteration;
    std::vector<std::uint32_t> ent(std::max<size_t>(predicted.size(), 1));
    std::uint32_t n = 0;
    throw_status(moeb_build_queue(predicted.data(), resident_mask.data(), static_cast<std::uint32_t>(predicted.size()),
                                  depth, ent.data(), &n));
    for (std::uint32_t i = 0; i < n; ++i) q.entries.push_back({ent[i], predicted[ent[i]], false});
    return q;
}

void clear_on_gate(PrefetchQueue& queue, std::uint32_t layer) {
    if (layer != queue.target_layer) throw std::logic_error("clear_on_gate: layer mismatch");
    std::erase_if(queue.entries, [](const PrefetchEntry& e) { return !e.issued; });
}

void PredictorStats::count_head(PredictedHeadKind kind, bool from_trace) {
    (from_trace ? trace_supplied : draws) += 1;
    if (kind == PredictedHeadKind::TopScore) ++head_top;
    else if (kind == PredictedHeadKind::ActiveNonTop) ++head_active;
    else ++head_inactive;
}

// ------------------------------------------------------------------ balancer
BalanceResult balance(const BalanceInput& input) {
    BalanceResult r;
    const std::uint32_t n = static_cast<std::uint32_t>(input.items.size());
    if (n == 0) return r;
    std::vector<std::uint32_t> uid(n), bat(n), ll(n), cl(n);
    for (std::uint32_t i = 0; i < n; ++i) {
        uid[i] = input.items[i].uid;
        bat[i] = input.items[i].batch;
    }
    std::uint32_t nl = 0, nc = 0;
    throw_status(moeb_balance(uid.data(), bat.data(), n, input.t_cpu_token, input.t_load, ll.data(), &nl, cl.data(),
                              &nc, &r.c_load, &r.c_cpu));
    r.load_list.assign(ll.begin(), ll.begin() + nl);
    r.cpu_list.assign(cl.begin(), cl.begin() + nc);
    return r;
}

TimeUnits brute_force_balance(const BalanceInput& input) {
    const std::size_t n = input.items.size();
    if (n > 20) throw ConfigError("brute_force_balance: too many items (max 20)");
    if (n == 0) return 0;
    TimeUnits best = ~TimeUnits{0};
    for (std::uint32_t m = 0; m < (1u << n); ++m) {
        TimeUnits lo = 0, cp = 0;
        for (std::size_t i = 0; i < n; ++i) {
            if (m >> i & 1u) lo += input.t_load;
            else cp += static_cast<TimeUnits>(input.items[i].batch) * input.t_cpu_token;
        }
        best = std::min(best, std::max(lo, cp));
    }
    return best;
}

}  // namespace moesched
