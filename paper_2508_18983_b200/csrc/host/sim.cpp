// sim.cpp — trace workload + decode-loop members of the moesched drop-in API.
// simulate() hands the whole trace to the device decision engine
// (moeb_simulate: the run_layer state machine in one persistent CTA) and
// converts the result to the reference's SimOutput. Trace I/O, the reuse
// curve and the timeline auditor are host utilities (reference behaviour:
// /root/reference/proj/src/trace.cpp:153-372, pipeline.cpp:374-531).
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <map>
#include <numeric>
#include <sstream>

#include "moesched/pipeline.hpp"
#include "moesched/router.hpp"
#include "moesched_b200.h"

namespace moesched {

void throw_status(int rc);

// --------------------------------------------------------------------- trace
GateTrace generate_trace(const ModelShape& shape, const SkewProfile& profile, std::uint64_t iterations,
                         std::uint64_t seed) {
    GateTrace tr;
    tr.shape = shape;
    const std::uint32_t L = shape.num_layers, E = shape.experts_per_layer, B = shape.batch_size;
    std::vector<double> flat((size_t)iterations * L * B * E);
    if (iterations)
        throw_status(moeb_generate_trace(L, E, B, profile.hot_fraction, profile.hot_mass, profile.persistence,
                                         profile.concentration, iterations, seed, flat.data()));
    size_t o = 0;
    for (std::uint64_t it = 0; it < iterations; ++it) {
        TraceIteration ti;
        ti.scores.resize(L);
        ti.predicted.resize(L);
        for (std::uint32_t l = 0; l < L; ++l) {
            ti.predicted[l].assign(B, {});
            for (std::uint32_t t = 0; t < B; ++t, o += E) ti.scores[l].emplace_back(flat.begin() + o, flat.begin() + o + E);
        }
        tr.iterations.push_back(std::move(ti));
    }
    return tr;
}

void save_trace(const GateTrace& trace, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open trace file for writing: " + path);
    const ModelShape& s = trace.shape;
    out << nlohmann::json{{"L", s.num_layers}, {"E", s.experts_per_layer}, {"k", s.top_k}, {"B", s.batch_size}}.dump()
        << '\n';
    for (std::uint64_t it = 0; it < trace.iterations.size(); ++it) {
        const TraceIteration& ti = trace.iterations[it];
        for (std::uint32_t l = 0; l < s.num_layers; ++l)
            for (std::uint32_t t = 0; t < s.batch_size; ++t) {
                nlohmann::json rec = {{"it", it}, {"layer", l}, {"tok", t}, {"s", ti.scores[l][t]}};
                if (!ti.predicted[l][t].empty()) rec["pred"] = ti.predicted[l][t];
                out << rec.dump() << '\n';
            }
    }
    if (!out) throw IoError("write failure on trace file: " + path);
}

GateTrace load_trace(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open trace file: " + path);
    auto fail = [&path](std::uint64_t n, const std::string& what) {
        std::ostringstream m;
        m << path << ":" << n << ": " << what;
        return IoError(m.str());
    };
    std::string line;
    std::uint64_t ln = 0;
    if (!std::getline(in, line)) throw fail(1, "missing header line");
    ++ln;
    GateTrace tr;
    try {
        const nlohmann::json h = nlohmann::json::parse(line);
        tr.shape.num_layers = h.at("L").get<std::uint32_t>();
        tr.shape.experts_per_layer = h.at("E").get<std::uint32_t>();
        tr.shape.top_k = h.at("k").get<std::uint32_t>();
        tr.shape.batch_size = h.at("B").get<std::uint32_t>();
    } catch (const nlohmann::json::exception& e) {
        throw fail(ln, std::string("bad header: ") + e.what());
    }
    const std::uint32_t L = tr.shape.num_layers, E = tr.shape.experts_per_layer, B = tr.shape.batch_size;
    if (L == 0 || E == 0 || B == 0) throw fail(ln, "header dimensions must be positive");
    auto fresh = [&] {
        TraceIteration ti;
        ti.scores.assign(L, std::vector<std::vector<double>>(B));
        ti.predicted.assign(L, std::vector<std::vector<double>>(B));
        return ti;
    };
    TraceIteration cur = fresh();
    std::uint64_t want_it = 0;
    std::uint32_t want_l = 0, want_t = 0;
    bool partial = false;
    while (std::getline(in, line)) {
        ++ln;
        if (line.empty()) continue;
        nlohmann::json rec;
        try {
            rec = nlohmann::json::parse(line);
        } catch (const nlohmann::json::exception& e) {
            throw fail(ln, std::string("malformed record: ") + e.what());
        }
        std::uint64_t it;
        std::uint32_t l, t;
        std::vector<double> s;
        try {
            it = rec.at("it").get<std::uint64_t>();
            l = rec.at("layer").get<std::uint32_t>();
            t = rec.at("tok").get<std::uint32_t>();
            s = rec.at("s").get<std::vector<double>>();
        } catch (const nlohmann::json::exception& e) {
            throw fail(ln, std::string("missing field: ") + e.what());
        }
        if (it != want_it || l != want_l || t != want_t) {
            std::ostringstream m;
            m << "record out of order: got (it=" << it << ", layer=" << l << ", tok=" << t << "), expected (it="
              << want_it << ", layer=" << want_l << ", tok=" << want_t << ")";
            throw fail(ln, m.str());
        }
        if (s.size() != E) {
            std::ostringstream m;
            m << "field 's': expected " << E << " scores, got " << s.size();
            throw fail(ln, m.str());
        }
        double sum = 0.0;
        for (double v : s) {
            if (v < 0.0) throw fail(ln, "field 's': negative score");
            sum += v;
        }
        if (sum > 1.0 + 1e-6) throw fail(ln, "field 's': scores sum above 1");
        cur.scores[l][t] = std::move(s);
        if (rec.contains("pred")) {
            std::vector<double> p;
            try {
                p = rec.at("pred").get<std::vector<double>>();
            } catch (const nlohmann::json::exception& e) {
                throw fail(ln, std::string("field 'pred': ") + e.what());
            }
            if (p.size() != E) {
                std::ostringstream m;
                m << "field 'pred': expected " << E << " scores, got " << p.size();
                throw fail(ln, m.str());
            }
            cur.predicted[l][t] = std::move(p);
        }
        partial = true;
        if (++want_t == B) {
            want_t = 0;
            if (++want_l == L) {
                want_l = 0;
                ++want_it;
                tr.iterations.push_back(std::move(cur));
                cur = fresh();
                partial = false;
            }
        }
    }
    if (partial || want_l != 0 || want_t != 0) throw fail(ln, "truncated trace: incomplete final iteration");
    return tr;
}

std::vector<double> reuse_curve(const GateTrace& trace) {
    if (trace.iterations.size() < 2) throw ConfigError("reuse_curve: needs >=2 iterations");
    const std::uint32_t E = trace.shape.experts_per_layer, k = trace.shape.top_k;
    std::vector<std::uint64_t> hits(E, 0);
    std::uint64_t samples = 0;
    auto rank = [E](const std::vector<double>& s) {  // score desc, index asc
        std::vector<std::uint32_t> o(E);
        std::iota(o.begin(), o.end(), 0u);
        std::stable_sort(o.begin(), o.end(), [&s](std::uint32_t a, std::uint32_t b) { return s[a] > s[b]; });
        return o;
    };
    for (size_t it = 0; it + 1 < trace.iterations.size(); ++it)
        for (std::uint32_t l = 0; l < trace.shape.num_layers; ++l)
            for (std::uint32_t t = 0; t < trace.shape.batch_size; ++t) {
                const auto now = rank(trace.iterations[it].scores[l][t]);
                const auto next = rank(trace.iterations[it + 1].scores[l][t]);
                std::vector<std::uint8_t> active(E, 0);
                for (std::uint32_t i = 0; i < k && i < E; ++i) active[next[i]] = 1;
                for (std::uint32_t r = 0; r < E; ++r) hits[r] += active[now[r]];
                ++samples;
            }
    std::vector<double> curve(E);
    for (std::uint32_t r = 0; r < E; ++r) curve[r] = static_cast<double>(hits[r]) / static_cast<double>(samples);
    return curve;
}

std::string fingerprint_bytes(const std::string& bytes) {
    std::uint64_t h = 0xcbf29ce484222325ULL;  // FNV-1a 64
    for (unsigned char c : bytes) {
        h ^= c;
        h *= 0x100000001b3ULL;
    }
    char buf[17];
    std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(h));
    return buf;
}

std::string fingerprint_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open file for fingerprinting: " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return fingerprint_bytes(ss.str());
}

// ------------------------------------------------------------------ pipeline
const char* to_string(Resource r) {
    switch (r) {
        case Resource::GPU: return "GPU";
        case Resource::CPU: return "CPU";
        case Resource::PCIE: return "PCIE";
    }
    return "?";
}

const char* to_string(TaskKind k) {
    static const char* kNames[] = {"Attn", "Route", "ResidentExpert", "LoadedExpert", "CpuExpert", "DemandLoad",
                                   "PrefetchLoad"};
    const auto i = static_cast<unsigned>(k);
    return i < 7 ? kNames[i] : "?";
}

// SimConfig (core.hpp:94-106) -> the C-ABI's flattened moeb_config.
moeb_config to_moeb_config(const SimConfig& cfg) {
    moeb_config c{};
    c.num_layers = cfg.shape.num_layers;
    c.experts = cfg.shape.experts_per_layer;
    c.top_k = cfg.shape.top_k;
    c.batch = cfg.shape.batch_size;
    c.alpha = cfg.router.alpha;
    c.slots = cfg.cache.slots_per_layer;
    c.window = cfg.cache.history_window;
    c.policy = cfg.cache.policy == CachePolicy::LRU ? 1 : 0;
    c.init_fill = cfg.cache.init_fill == InitFill::FirstSlots ? 0 : cfg.cache.init_fill == InitFill::SeededRandom ? 1 : 2;
    c.t_attn = cfg.cost.t_attn;
    c.t_gpu = cfg.cost.t_gpu;
    c.t_cpu_token = cfg.cost.t_cpu_token;
    c.t_load = cfg.cost.t_load;
    c.t_route = cfg.cost.t_route;
    c.p_top = cfg.predictor.p_top;
    c.p_active = cfg.predictor.p_active;
    c.queue_depth = cfg.predictor.queue_depth;
    c.ce = cfg.stages.ce;
    c.er = cfg.stages.er;
    c.pre = cfg.stages.pre;
    c.ba = cfg.stages.ba;
    c.seed = cfg.seed;
    return c;
}

SimOutput simulate(const GateTrace& trace, const SimConfig& cfg) {
    const ValidationReport rep = validate_config(cfg);
    if (!rep.ok())
        throw ConfigError("invalid config: " + rep.violations.front().field + ": " + rep.violations.front().rule);
    if (!(trace.shape == cfg.shape)) throw ConfigError("trace shape does not match config shape");
    const ModelShape& s = cfg.shape;
    const std::uint32_t L = s.num_layers, E = s.experts_per_layer, B = s.batch_size;
    const std::uint64_t iters = trace.iterations.size();
    std::vector<double> scores((size_t)iters * L * B * E), pred;
    std::vector<std::uint8_t> has;
    bool any_pred = false;
    for (const TraceIteration& ti : trace.iterations)
        for (const auto& layer : ti.predicted)
            for (const auto& v : layer) any_pred |= !v.empty();
    if (any_pred) {
        pred.assign(scores.size(), 0.0);
        has.assign((size_t)iters * L * B, 0);
    }
    size_t row = 0;
    for (const TraceIteration& ti : trace.iterations)
        for (std::uint32_t l = 0; l < L; ++l)
            for (std::uint32_t t = 0; t < B; ++t, ++row) {
                std::copy(ti.scores[l][t].begin(), ti.scores[l][t].end(), scores.begin() + row * E);
                if (any_pred && !ti.predicted[l][t].empty()) {
                    std::copy(ti.predicted[l][t].begin(), ti.predicted[l][t].end(), pred.begin() + row * E);
                    has[row] = 1;
                }
            }
    const moeb_config c = to_moeb_config(cfg);
    moeb_result* r = nullptr;
    throw_status(moeb_simulate(&c, scores.data(), any_pred ? pred.data() : nullptr, any_pred ? has.data() : nullptr,
                               iters, 0, &r));
    SimOutput out;
    moeb_metrics m{};
    moeb_result_metrics(r, &m);
    out.metrics.stage = cfg.stages.label();
    out.metrics.tpot = m.tpot;
    out.metrics.hit_rate = m.hit_rate;
    out.metrics.substitution_ratio = m.substitution_ratio;
    out.metrics.demand_loads = m.demand_loads;
    out.metrics.prefetch_loads = m.prefetch_loads;
    out.metrics.cpu_computed = m.cpu_computed;
    out.metrics.hits = m.hits;
    out.metrics.misses = m.misses;
    out.metrics.substitutions = m.substitutions;
    out.metrics.low_score_kept = m.low_score_kept;
    out.metrics.selections = m.selections;
    out.metrics.iterations = m.iterations;
    out.metrics.total_time = m.total_time;
    out.prefetch_stats = PredictorStats{m.draws, m.trace_supplied, m.head_top, m.head_active, m.head_inactive,
                                        m.issued, m.cancelled};
    const moeb_task* tasks;
    size_t n;
    moeb_result_tasks(r, &tasks, &n);
    for (size_t i = 0; i < n; ++i) {
        Task t;
        t.resource = static_cast<Resource>(tasks[i].resource);
        t.kind = static_cast<TaskKind>(tasks[i].kind);
        if (tasks[i].expert_layer >= 0) t.expert = ExpertId{static_cast<std::uint32_t>(tasks[i].expert_layer), tasks[i].expert};
        t.start = tasks[i].start;
        t.end = tasks[i].end;
        t.layer = tasks[i].layer;
        t.iteration = tasks[i].iteration;
        out.timeline.tasks.push_back(t);
    }
    const moeb_window* w;
    moeb_result_windows(r, &w, &n);
    for (size_t i = 0; i < n; ++i) {
        LayerWindow lw{w[i].iteration, w[i].layer, w[i].attn_end, w[i].route_end, w[i].completion, {}};
        for (std::uint32_t e = 0; e < 64; ++e)
            if (w[i].selected >> e & 1ULL) lw.selected.push_back(e);
        out.timeline.windows.push_back(std::move(lw));
    }
    const moeb_eviction* ev;
    moeb_result_evictions(r, &ev, &n);
    for (size_t i = 0; i < n; ++i) out.timeline.evictions.push_back({ev[i].time, ev[i].layer, ev[i].expert});
    const std::uint64_t* itc;
    moeb_result_iteration_completion(r, &itc, &n);
    out.timeline.iteration_completion.assign(itc, itc + n);
    std::vector<std::uint32_t> buf(E + 1);
    for (std::uint32_t l = 0; l < L; ++l) {
        std::uint32_t k = 0;
        moeb_result_cache_final(r, l, buf.data(), &k);
        out.cache_final.emplace_back(buf.begin(), buf.begin() + k);
    }
    moeb_result_free(r);
    return out;
}

std::vector<SimOutput> run_ablation(const GateTrace& trace, const SimConfig& base) {
    static const StageSet kLadder[] = {{false, false, false, false}, {true, false, false, false},
                                       {true, true, false, false},   {true, true, true, false},
                                       {true, true, true, true}};
    std::vector<SimOutput> runs;
    for (const StageSet& st : kLadder) {
        SimConfig c = base;
        c.stages = st;
        runs.push_back(simulate(trace, c));
    }
    return runs;
}

// The invariant auditor (test-side tool of the reference, pipeline.cpp:405-531).
std::vector<std::string> verify_timeline(const Timeline& tl) {
    std::vector<std::string> bad;
    for (int ri = 0; ri < 3; ++ri) {
        const Resource res = static_cast<Resource>(ri);
        std::vector<const Task*> ts;
        for (const Task& t : tl.tasks)
            if (t.resource == res) ts.push_back(&t);
        std::sort(ts.begin(), ts.end(), [](const Task* a, const Task* b) {
            return a->start != b->start ? a->start < b->start : a->end < b->end;
        });
        for (size_t i = 0; i < ts.size(); ++i) {
            if (ts[i]->end < ts[i]->start) {
                std::ostringstream m;
                m << to_string(res) << " task ends before it starts at t=" << ts[i]->start;
                bad.push_back(m.str());
            }
            if (i > 0 && ts[i]->start < ts[i - 1]->end) {
                std::ostringstream m;
                m << to_string(res) << " tasks overlap: [" << ts[i - 1]->start << ", " << ts[i - 1]->end << ") and ["
                  << ts[i]->start << ", " << ts[i]->end << ")";
                bad.push_back(m.str());
            }
        }
    }
    for (const Task& t : tl.tasks) {
        Resource want = Resource::GPU;
        if (t.kind == TaskKind::Route || t.kind == TaskKind::CpuExpert) want = Resource::CPU;
        if (t.kind == TaskKind::DemandLoad || t.kind == TaskKind::PrefetchLoad) want = Resource::PCIE;
        if (t.resource != want) bad.push_back(std::string(to_string(t.kind)) + " scheduled on " + to_string(t.resource));
    }
    for (const Task& t : tl.tasks) {
        if (t.kind != TaskKind::LoadedExpert || !t.expert) continue;
        const Task* load = nullptr;
        for (const Task& d : tl.tasks)
            if (d.kind == TaskKind::DemandLoad && d.iteration == t.iteration && d.layer == t.layer && d.expert == t.expert) {
                load = &d;
                break;
            }
        std::ostringstream m;
        m << "LoadedExpert (" << t.expert->layer << "," << t.expert->index << ")";
        if (!load) bad.push_back(m.str() + " has no matching DemandLoad");
        else if (load->end > t.start) {
            m << " starts at " << t.start << " before its load ends at " << load->end;
            bad.push_back(m.str());
        }
    }
    for (const LayerWindow& w : tl.windows)
        for (const EvictionEvent& e : tl.evictions) {
            if (e.layer != w.layer || e.time < w.route_end || e.time >= w.completion) continue;
            if (std::binary_search(w.selected.begin(), w.selected.end(), e.expert)) {
                std::ostringstream m;
                m << "expert (" << w.layer << "," << e.expert << ") evicted at t=" << e.time
                  << " while selected in iteration " << w.iteration;
                bad.push_back(m.str());
            }
        }
    for (const Task& d : tl.tasks) {
        if (d.kind != TaskKind::DemandLoad) continue;
        TimeUnits ready = d.start;
        for (const LayerWindow& w : tl.windows)
            if (w.iteration == d.iteration && w.layer == d.layer) {
                ready = w.route_end;
                break;
            }
        if (d.start <= ready) continue;
        for (const Task& p : tl.tasks)
            if (p.kind == TaskKind::PrefetchLoad && p.start >= ready && p.start < d.start && p.end > ready) {
                std::ostringstream m;
                m << "DemandLoad at t=" << d.start << " (ready " << ready << ") waited behind PrefetchLoad dispatched at t="
                  << p.start;
                bad.push_back(m.str());
            }
    }
    return bad;
}

}  // namespace moesched
