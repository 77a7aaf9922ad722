// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A small extern "C" driver over the UNMODIFIED reference library, compiled
// from the sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libmoesched_ref.so. Python tests and tests/golden/make_golden.py
// call it through ctypes to (a) pin the C restatement in
// oracle/moesched_oracle.c and (b) emit golden decision dumps. The JSON
// schema matches orc_simulate_json() so the two can be compared directly.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "moesched/balancer.hpp"
#include "moesched/cache.hpp"
#include "moesched/pipeline.hpp"
#include "moesched/prefetch.hpp"
#include "moesched/report.hpp"
#include "moesched/router.hpp"
#include "moesched/trace.hpp"

#include "moesched_oracle.h"  // only for the orc_config struct layout

using namespace moesched;

namespace {

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

std::string num(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

template <class V>
std::string list(const V& v) {
  std::string s = "[";
  for (std::size_t i = 0; i < v.size(); ++i) {
    if (i) s += ",";
    s += std::to_string(v[i]);
  }
  return s + "]";
}

SimConfig to_cfg(const orc_config* c) {
  SimConfig cfg;
  cfg.shape = {c->num_layers, c->experts, c->top_k, c->batch};
  cfg.router.alpha = c->alpha;
  cfg.cache.slots_per_layer = c->slots;
  cfg.cache.history_window = c->window;
  cfg.cache.policy = c->policy == 0 ? CachePolicy::ScoreWindow : CachePolicy::LRU;
  cfg.cache.init_fill = c->init_fill == 0   ? InitFill::FirstSlots
                        : c->init_fill == 1 ? InitFill::SeededRandom
                                            : InitFill::Empty;
  cfg.cost = {c->t_attn, c->t_gpu, c->t_cpu_token, c->t_load, c->t_route};
  cfg.predictor = {c->p_top, c->p_active, c->queue_depth};
  cfg.stages = {c->ce != 0, c->er != 0, c->pre != 0, c->ba != 0};
  cfg.seed = c->seed;
  return cfg;
}

GateTrace to_trace(const orc_config* c, const double* scores, const double* pred,
                   const std::uint8_t* has_pred, std::uint64_t iters) {
  GateTrace tr;
  tr.shape = {c->num_layers, c->experts, c->top_k, c->batch};
  const std::size_t E = c->experts;
  for (std::uint64_t it = 0; it < iters; ++it) {
    TraceIteration ti;
    ti.scores.resize(c->num_layers);
    ti.predicted.resize(c->num_layers);
    for (std::uint32_t l = 0; l < c->num_layers; ++l) {
      for (std::uint32_t t = 0; t < c->batch; ++t) {
        const std::size_t row = (it * c->num_layers + l) * c->batch + t;
        ti.scores[l].emplace_back(scores + row * E, scores + (row + 1) * E);
        if (pred && has_pred && has_pred[row]) {
          ti.predicted[l].emplace_back(pred + row * E, pred + (row + 1) * E);
        } else {
          ti.predicted[l].emplace_back();
        }
      }
    }
    tr.iterations.push_back(std::move(ti));
  }
  return tr;
}

std::string sim_json(const SimOutput& out, bool timeline) {
  const Metrics& m = out.metrics;
  std::ostringstream j;
  j << "{\"metrics\":{\"tpot\":" << num(m.tpot) << ",\"hit_rate\":" << num(m.hit_rate)
    << ",\"substitution_ratio\":" << num(m.substitution_ratio)
    << ",\"demand_loads\":" << m.demand_loads << ",\"prefetch_loads\":" << m.prefetch_loads
    << ",\"cpu_computed\":" << m.cpu_computed << ",\"hits\":" << m.hits
    << ",\"misses\":" << m.misses << ",\"substitutions\":" << m.substitutions
    << ",\"low_score_kept\":" << m.low_score_kept << ",\"selections\":" << m.selections
    << ",\"iterations\":" << m.iterations << ",\"total_time\":" << m.total_time << "},";
  const PredictorStats& s = out.prefetch_stats;
  j << "\"stats\":{\"draws\":" << s.draws << ",\"trace_supplied\":" << s.trace_supplied
    << ",\"head_top\":" << s.head_top << ",\"head_active\":" << s.head_active
    << ",\"head_inactive\":" << s.head_inactive << ",\"issued\":" << s.issued
    << ",\"cancelled\":" << s.cancelled << "},";
  j << "\"cache_final\":[";
  for (std::size_t l = 0; l < out.cache_final.size(); ++l) j << (l ? "," : "") << list(out.cache_final[l]);
  j << "]";
  if (timeline) {
    const Timeline& tl = out.timeline;
    std::vector<std::tuple<std::uint64_t, int, std::uint64_t, std::uint32_t, std::uint64_t, int, int,
                           std::uint32_t>>
        keyed;
    for (const Task& t : tl.tasks) {
      keyed.emplace_back(t.start, static_cast<int>(t.resource), t.end, t.layer, t.iteration,
                         static_cast<int>(t.kind), t.expert ? static_cast<int>(t.expert->layer) : -1,
                         t.expert ? t.expert->index : 0u);
    }
    std::sort(keyed.begin(), keyed.end());
    j << ",\"tasks\":[";
    for (std::size_t i = 0; i < keyed.size(); ++i) {
      const auto& [st, res, en, layer, it, kind, el, ei] = keyed[i];
      j << (i ? "," : "") << "[" << res << "," << kind << "," << el << "," << ei << "," << st << ","
        << en << "," << layer << "," << it << "]";
    }
    j << "],\"windows\":[";
    for (std::size_t i = 0; i < tl.windows.size(); ++i) {
      const LayerWindow& w = tl.windows[i];
      j << (i ? "," : "") << "[" << w.iteration << "," << w.layer << "," << w.attn_end << ","
        << w.route_end << "," << w.completion << "," << list(w.selected) << "]";
    }
    j << "],\"evictions\":[";
    for (std::size_t i = 0; i < tl.evictions.size(); ++i) {
      const EvictionEvent& e = tl.evictions[i];
      j << (i ? "," : "") << "[" << e.time << "," << e.layer << "," << e.expert << "]";
    }
    j << "],\"iteration_completion\":" << list(tl.iteration_completion);
  }
  j << "}";
  return j.str();
}

}  // namespace

extern "C" {

char* ref_simulate_json(const orc_config* c, const double* scores, const double* pred,
                        const std::uint8_t* has_pred, std::uint64_t iters, int emit_timeline) {
  try {
    const GateTrace tr = to_trace(c, scores, pred, has_pred, iters);
    const SimOutput out = simulate(tr, to_cfg(c));
    const std::vector<std::string> v = verify_timeline(out.timeline);
    std::string j = sim_json(out, emit_timeline != 0);
    j.pop_back();
    j += ",\"timeline_violations\":" + std::to_string(v.size()) + "}";
    return dup(j);
  } catch (const std::exception& e) {
    return dup(std::string("{\"error\":\"") + e.what() + "\"}");
  }
}

// Wall time (ns) of the reference's simulate() alone on a trace — the CPU
// decision path's cost, without verify_timeline (an O(N^2) test auditor) or
// the JSON marshalling. Returns 0 on error.
std::uint64_t ref_simulate_ns(const orc_config* c, const double* scores, std::uint64_t iters) {
  try {
    const GateTrace tr = to_trace(c, scores, nullptr, nullptr, iters);
    const SimConfig cfg = to_cfg(c);
    const auto t0 = std::chrono::steady_clock::now();
    const SimOutput out = simulate(tr, cfg);
    const auto t1 = std::chrono::steady_clock::now();
    if (out.metrics.iterations != iters) return 0;
    return (std::uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
  } catch (const std::exception&) {
    return 0;
  }
}

// route (+ optional coalesce) on one batch; JSON with per-token records.
char* ref_route_json(const double* scores, std::uint32_t B, std::uint32_t E,
                     const std::uint8_t* mask, std::uint32_t k, double alpha, int coalesce) {
  try {
    std::vector<std::vector<double>> batch;
    for (std::uint32_t t = 0; t < B; ++t) batch.emplace_back(scores + t * E, scores + (t + 1) * E);
    std::span<const std::uint8_t> m(mask, E);
    RouteResult r = route(batch, m, k, alpha);
    if (coalesce) r = coalesce_for_batching(r, batch, m);
    std::ostringstream j;
    j << "{\"C\":" << list(r.top_score_set) << ",\"pending\":" << list(r.pending) << ",\"tok\":[";
    for (std::size_t t = 0; t < r.tokens.size(); ++t) {
      const TokenRoute& tk = r.tokens[t];
      j << (t ? "," : "") << "{\"sel\":" << list(tk.selected) << ",\"sub\":[";
      for (std::size_t i = 0; i < tk.substitutions.size(); ++i)
        j << (i ? "," : "") << "[" << tk.substitutions[i].dropped << "," << tk.substitutions[i].chosen << "]";
      j << "],\"kept\":" << list(tk.kept_low) << ",\"beta\":" << num(tk.cls.beta)
        << ",\"actives\":" << list(tk.cls.actives) << ",\"top\":" << list(tk.cls.top_score)
        << ",\"low\":" << list(tk.cls.low_score) << ",\"alt\":" << list(tk.cls.alt_band) << "}";
    }
    j << "]}";
    return dup(j.str());
  } catch (const std::exception& e) {
    return dup(std::string("{\"error\":\"") + e.what() + "\"}");
  }
}

void ref_generate_trace(std::uint32_t L, std::uint32_t E, std::uint32_t k, std::uint32_t B,
                        double hot_fraction, double hot_mass, double persistence,
                        double concentration, std::uint64_t iters, std::uint64_t seed,
                        double* out) {
  SkewProfile p{hot_fraction, hot_mass, persistence, concentration};
  const GateTrace tr = generate_trace({L, E, k, B}, p, iters, seed);
  std::size_t o = 0;
  for (const auto& it : tr.iterations)
    for (const auto& layer : it.scores)
      for (const auto& v : layer)
        for (double s : v) out[o++] = s;
}

// Times simulate() (decision path only, one thread) over the trace; returns
// seconds for `reps` runs.
double ref_time_simulate(const orc_config* c, const double* scores, std::uint64_t iters, int reps) {
  const GateTrace tr = to_trace(c, scores, nullptr, nullptr, iters);
  const SimConfig cfg = to_cfg(c);
  const auto t0 = std::chrono::steady_clock::now();
  std::uint64_t sink = 0;
  for (int r = 0; r < reps; ++r) sink += simulate(tr, cfg).metrics.hits;
  const auto t1 = std::chrono::steady_clock::now();
  if (sink == 0xffffffffffffULL) std::puts("");
  return std::chrono::duration<double>(t1 - t0).count();
}

// The reference's own JSONL loader (with its validation) + simulate() +
// build_report() on a trace file: the receiving side of the wire-format
// bridge (paper_2508_18983_b200/bridge.py).
char* ref_report_from_trace_file(const orc_config* c, const char* path) {
  try {
    const GateTrace tr = load_trace(path);
    const SimOutput out = simulate(tr, to_cfg(c));
    return dup(build_report(to_cfg(c), out, fingerprint_file(path)).dump());
  } catch (const std::exception& e) {
    return dup(std::string("{\"error\":\"") + e.what() + "\"}");
  }
}

void ref_free(void* p) { std::free(p); }

}  // extern "C"
