// engine_kernels.cu — decision-engine kernels and the decision-path C-ABI.
//
// Kernels:
//   replay_kernel     simulate() (pipeline.cpp:374-385): the whole
//                     run_layer/schedule_prefetch loop over a score trace in
//                     ONE persistent CTA (no host round trip per step).
//   route_kernel      route / coalesce_for_batching (router.cpp:97-260)
//   classify_kernel   classify / plain_top_k (router.cpp:35-71)
//   balance_kernel    balance (balancer.cpp:8-38)
//   predict_kernel    predict_scores (prefetch.cpp:34-83)
//   queue_kernel      build_queue (prefetch.cpp:85-115)
//   cache_op_kernel   CacheState members (cache.cpp:10-165)
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/moesched_b200.h"
#include "decide.cuh"
#include "engine_host.h"
#include "host_common.h"

namespace moeb {

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

// =================================================================== kernels

struct ReplayArgs {
  DevCfg cfg;
  EngineState* st;
  LayerState* layers;
  double* hist;
  const double* scores;   // [iters][L][B][E]
  const double* pred;     // nullable
  const uint8_t* has_pred;
  uint64_t iters;
  Logs logs;
  int32_t record_steps;
};

struct ReplaySmem {
  DecideSmem d;
  NextSmem n;
  StepScratch s;
  DevCfg cfg;
};

__global__ void __launch_bounds__(kThreads, 1) replay_kernel(ReplayArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ReplaySmem* sm = reinterpret_cast<ReplaySmem*>(smem_raw);
  if (threadIdx.x == 0) sm->cfg = a.cfg;
  __syncthreads();
  const DevCfg& cfg = sm->cfg;
  const uint32_t L = cfg.L, B = cfg.B, E = cfg.E;
  const size_t step_elems = (size_t)B * E;
  uint64_t step_idx = 0;
  for (uint64_t it = 0; it < a.iters; ++it) {
    for (uint32_t layer = 0; layer < L; ++layer, ++step_idx) {
      const double* src = a.scores + ((size_t)it * L + layer) * step_elems;
      for (uint32_t i = threadIdx.x; i < step_elems; i += blockDim.x)
        sm->d.s[i / E][i % E] = src[i];
      StepCtx cx;
      cx.cfg = &cfg;
      cx.st = a.st;
      uint64_t tit = it;
      uint32_t tl = layer + 1;
      if (tl == L) { tl = 0; ++tit; }
      cx.ls = &a.layers[layer];
      cx.hist_l = a.hist + (size_t)layer * cfg.window * E;
      cx.tls = &a.layers[tl];
      cx.thist = a.hist + (size_t)tl * cfg.window * E;
      cx.logs = &a.logs;
      cx.prof = nullptr;
      cx.it = it;
      cx.layer = layer;
      cx.has_target = tit < a.iters;
      cx.target_layer = tl;
      cx.target_it = tit;
      cx.defer_prefetch = 0;
      cx.f32_scores = 0;
      cx.run_pending = 0;
      cx.prev_rec = nullptr;
      if (cfg.pre && cx.has_target) {
        const size_t row0 = ((size_t)tit * L + tl) * B;
        const double* ns = a.scores + row0 * E;
        for (uint32_t i = threadIdx.x; i < step_elems; i += blockDim.x) {
          sm->d.ns[i / E][i % E] = ns[i];
          sm->d.np[i / E][i % E] = a.pred ? a.pred[row0 * E + i] : 0.0;
        }
        if (threadIdx.x == 0) {
          uint64_t m = 0;
          if (a.pred && a.has_pred)
            for (uint32_t t = 0; t < B; ++t) m |= (uint64_t)(a.has_pred[row0 + t] != 0) << t;
          sm->d.next_has_pred = m;
        }
      }
      __syncthreads();
      StepRec* rec = nullptr;
      TokRec* toks = nullptr;
      if (a.record_steps && a.logs.steps && step_idx < a.logs.cap_steps) {
        rec = a.logs.steps + step_idx;
        toks = a.logs.toks + step_idx * B;
      }
      decide_step(cx, &sm->d, &sm->n, &sm->s, rec, toks);
      __syncthreads();
      if (a.st->err) return;
    }
  }
}

// ---- library-level single calls

struct RouteIO {
  uint8_t sel[kMaxB][kMaxK], sub_d[kMaxB][kMaxK], sub_c[kMaxB][kMaxK], kept[kMaxB][kMaxK];
  uint8_t nsel[kMaxB], nsub[kMaxB], nkept[kMaxB];
  uint64_t C;
  uint64_t pending;
  // mode 2: the caller's per-token thresholds {beta, T, L, R} (the bands a
  // RouteResult was classified with); classify outputs for token 0 (mode 3/4)
  double thr_tok[kMaxB][4];
  double thr[4];
  uint8_t order[kMaxE];
  uint64_t act, top, low, alt;
};

// mode 0: route, 1: route + coalesce, 2: coalesce an existing result (io in),
// 3: classify only, 4: plain top-k
__global__ void __launch_bounds__(kThreads, 1) route_kernel(const double* scores, uint32_t B,
                                                            uint32_t E, uint64_t resident,
                                                            uint32_t k, double alpha, int mode,
                                                            RouteIO* io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ReplaySmem* sm = reinterpret_cast<ReplaySmem*>(smem_raw);
  DecideSmem* d = &sm->d;
  const int warp = warp_id(), lane = lane_id();
  for (uint32_t i = threadIdx.x; i < B * E; i += blockDim.x) d->s[i / E][i % E] = scores[i];
  __syncthreads();
  for (uint32_t t = warp; t < B; t += kWarps) {
    uint64_t a, tp, lw, al;
    double b, T, Lb, R;
    classify_warp(d->s[t], E, k, alpha, d->order[t], a, tp, lw, al, b, T, Lb, R);
    if (lane == 0) {
      d->act[t] = a; d->top[t] = tp; d->low[t] = lw; d->alt[t] = al;
      d->beta[t] = b; d->thT[t] = T; d->thL[t] = Lb; d->thR[t] = R;
    }
  }
  __syncthreads();
  if (mode == 2) {
    // re-derive the bands from the given thresholds, exactly as classified
    for (uint32_t t = warp; t < B; t += kWarps) {
      const double b = io->thr_tok[t][0], T = io->thr_tok[t][1], Lb = io->thr_tok[t][2], R = io->thr_tok[t][3];
      bool l0 = false, l1 = false, a0 = false, a1 = false;
      const uint32_t e0 = lane, e1 = lane + 32;
      if (e0 < E) { const double s0 = d->s[t][e0]; l0 = has(d->act[t], e0) && b > 0.0 && s0 >= Lb && s0 < T; a0 = !has(d->act[t], e0) && b > 0.0 && s0 >= R && s0 < Lb; }
      if (e1 < E) { const double s1 = d->s[t][e1]; l1 = has(d->act[t], e1) && b > 0.0 && s1 >= Lb && s1 < T; a1 = !has(d->act[t], e1) && b > 0.0 && s1 >= R && s1 < Lb; }
      const uint64_t low = ballot64(l0, l1), alt = ballot64(a0, a1);
      if (lane == 0) {
        d->low[t] = low; d->alt[t] = alt; d->top[t] = d->act[t] & ~low;
        d->beta[t] = b; d->thT[t] = T; d->thL[t] = Lb; d->thR[t] = R;
      }
    }
    __syncthreads();
  }
  if (mode == 3 || mode == 4) {
    if (threadIdx.x == 0) {
      io->thr[0] = d->beta[0]; io->thr[1] = d->thT[0]; io->thr[2] = d->thL[0]; io->thr[3] = d->thR[0];
      io->act = d->act[0]; io->top = d->top[0]; io->low = d->low[0]; io->alt = d->alt[0];
    }
    for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) io->order[e] = d->order[0][e];
    return;
  }
  if (threadIdx.x == 0) {
    if (mode == 2) {
      d->C = io->C;
    } else {
      uint64_t C = 0;
      for (uint32_t t = 0; t < B; ++t) C |= d->top[t];
      d->C = C;
    }
  }
  __syncthreads();
  for (uint32_t t = warp; t < B; t += kWarps) {
    if (mode == 2) {
      if (lane != 0) continue;
      d->nsel[t] = io->nsel[t]; d->nsub[t] = io->nsub[t]; d->nkept[t] = io->nkept[t];
      for (int i = 0; i < kMaxK; ++i) {
        d->sel[t][i] = io->sel[t][i]; d->sub_d[t][i] = io->sub_d[t][i];
        d->sub_c[t][i] = io->sub_c[t][i]; d->kept[t][i] = io->kept[t][i];
      }
    } else {
      route_token_warp(d, t, resident, E, k, d->C);
    }
  }
  __syncthreads();
  if (warp == 0 && mode >= 1) coalesce_warp(d, B, E, k, resident, sm->s.cnt);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t pend = 0;
    for (uint32_t t = 0; t < B; ++t)
      for (uint32_t i = 0; i < d->nkept[t]; ++i)
        if (!has(resident, d->kept[t][i])) pend |= bit(d->kept[t][i]);
    io->pending = pend;
    io->C = d->C;
  }
  for (uint32_t t = threadIdx.x; t < B; t += blockDim.x) {
    io->nsel[t] = d->nsel[t]; io->nsub[t] = d->nsub[t]; io->nkept[t] = d->nkept[t];
    for (int i = 0; i < kMaxK; ++i) {
      io->sel[t][i] = d->sel[t][i]; io->sub_d[t][i] = d->sub_d[t][i];
      io->sub_c[t][i] = d->sub_c[t][i]; io->kept[t][i] = d->kept[t][i];
    }
  }
}

struct BalanceIO {
  uint8_t uid[kMaxE];
  uint16_t batch[kMaxE];
  uint32_t n;
  uint8_t load[kMaxE], cpu[kMaxE];
  uint32_t n_load, n_cpu;
};

__global__ void balance_kernel(BalanceIO* io, uint64_t t_cpu_token, uint64_t t_load) {
  __shared__ uint8_t uid[kMaxE];
  __shared__ uint16_t bat[kMaxE];
  __shared__ uint8_t ld[kMaxE], cp[kMaxE];
  for (uint32_t i = threadIdx.x; i < io->n; i += 32) { uid[i] = io->uid[i]; bat[i] = io->batch[i]; }
  __syncwarp();
  uint32_t nl, nc;
  balance_warp(uid, bat, io->n, t_cpu_token, t_load, ld, nl, cp, nc);
  if (threadIdx.x == 0) {
    io->n_load = nl;
    io->n_cpu = nc;
    for (uint32_t i = 0; i < nl; ++i) io->load[i] = ld[i];
    for (uint32_t i = 0; i < nc; ++i) io->cpu[i] = cp[i];
  }
}

// predict_scores on a single token: reuse the engine's prefetch code path by
// running decide-free pieces here (classify + head draw + swap).
struct PredictIO {
  double tn[kMaxE], sup[kMaxE], out[kMaxE];
  uint64_t rng[4];
  uint32_t head;
  int32_t kind;
  int32_t supplied;
};

__global__ void predict_kernel(PredictIO* io, uint32_t E, uint32_t k, double alpha, double p_top,
                               double p_active) {
  __shared__ uint8_t order[kMaxE];
  __shared__ double tn[kMaxE];
  const int lane = lane_id();
  for (uint32_t e = lane; e < E; e += 32) tn[e] = io->tn[e];
  __syncwarp();
  uint64_t act, top, low, alt;
  double b, T, L, R;
  classify_warp(tn, E, k, alpha, order, act, top, low, alt, b, T, L, R);
  auto argmax_first = [&](const double* v) -> uint32_t {
    double bv = 0.0;
    uint32_t bi = 0xffffffffu;
    for (uint32_t e = lane; e < E; e += 32)
      if (bi == 0xffffffffu || v[e] > bv) { bv = v[e]; bi = e; }
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const uint32_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (i2 != 0xffffffffu && (bi == 0xffffffffu || v2 > bv || (v2 == bv && i2 < bi))) { bv = v2; bi = i2; }
    }
    return bi;
  };
  uint32_t head;
  int kind;
  if (io->supplied) {
    head = argmax_first(io->sup);
    kind = has(top, head) ? 0 : (has(act, head) ? 1 : 2);
    for (uint32_t e = lane; e < E; e += 32) io->out[e] = io->sup[e];
  } else {
    uint64_t rs[4] = {io->rng[0], io->rng[1], io->rng[2], io->rng[3]};
    const uint32_t n_top = __popcll(top);
    if (rng_double(rs) < p_top && n_top > 0) {
      const uint32_t pick = (uint32_t)rng_below(rs, n_top);
      uint32_t c = 0;
      head = 0;
      for (uint32_t r = 0; r < k; ++r) {
        const uint32_t e = order[r];
        if (has(top, e)) { if (c == pick) { head = e; break; } ++c; }
      }
      kind = 0;
    } else {
      const uint64_t lows = act & ~top;
      const uint32_t n_low = __popcll(lows);
      if (rng_double(rs) < p_active && n_low > 0) {
        const uint32_t pick = (uint32_t)rng_below(rs, n_low);
        uint32_t c = 0;
        head = 0;
        for (uint32_t r = 0; r < k; ++r) {
          const uint32_t e = order[r];
          if (has(lows, e)) { if (c == pick) { head = e; break; } ++c; }
        }
        kind = 1;
      } else {
        const uint64_t allm = E >= 64 ? ~0ULL : ((1ULL << E) - 1ULL);
        const uint64_t inact = allm & ~act;
        const uint32_t pick = (uint32_t)rng_below(rs, __popcll(inact));
        uint64_t m = inact;
        for (uint32_t i = 0; i < pick; ++i) m &= m - 1;
        head = __ffsll((long long)m) - 1;
        kind = 2;
      }
    }
    const uint32_t tt = argmax_first(tn);
    for (uint32_t e = lane; e < E; e += 32)
      io->out[e] = (e == head) ? tn[tt] : ((e == tt) ? tn[head] : tn[e]);
    if (lane == 0) for (int i = 0; i < 4; ++i) io->rng[i] = rs[i];
  }
  if (lane == 0) { io->head = head; io->kind = kind; }
}

struct QueueIO {
  double pred[kMaxE];
  uint64_t mask;
  uint8_t ent[kMaxE];
  uint32_t n;
};

__global__ void queue_kernel(QueueIO* io, uint32_t E, uint32_t depth) {
  __shared__ uint8_t qorder[kMaxE];
  const int lane = lane_id();
  for (uint32_t e = lane; e < E; e += 32) {
    const double v = io->pred[e];
    uint32_t r = 0;
    for (uint32_t j = 0; j < E; ++j) {
      const double vj = io->pred[j];
      r += (vj > v) || (vj == v && j < e);
    }
    qorder[r] = (uint8_t)e;
  }
  __syncwarp();
  if (lane == 0) {
    uint32_t n = 0;
    for (uint32_t r = 0; r < E && n < depth; ++r)
      if (!has(io->mask, qorder[r])) io->ent[n++] = qorder[r];
    io->n = n;
  }
}

// ---- CacheState members, one op per launch (warp 0)
enum CacheOp : int32_t {
  OP_RECORD = 0, OP_AVG, OP_EVICT, OP_SHIELD, OP_UNSHIELD, OP_TOUCH, OP_ADMIT
};
struct CacheIO {
  double v[kMaxE];
  double out_d;
  int64_t out_i;
  int32_t rc;
};

__global__ void cache_op_kernel(DevCfg cfg, LayerState* layers, double* hist, int32_t op,
                                uint32_t layer, uint32_t e, uint64_t now, CacheIO* io) {
  LayerState* ls = &layers[layer];
  double* hist_l = hist + (size_t)layer * cfg.window * cfg.E;
  const int lane = lane_id();
  switch (op) {
    case OP_RECORD: record_scores_warp(ls, hist_l, cfg.window, cfg.E, io->v); break;
    case OP_AVG: {
      const double a = window_average(ls, hist_l, cfg.window, cfg.E, e);
      if (lane == 0) io->out_d = a;
      break;
    }
    case OP_EVICT: {
      const int v = try_evict_warp(ls, hist_l, cfg);
      if (lane == 0) io->out_i = v;
      break;
    }
    case OP_SHIELD: if (lane == 0) ls->shield |= bit(e); break;
    case OP_UNSHIELD: if (lane == 0) ls->shield = 0; break;
    case OP_TOUCH: if (lane == 0) ls->last_access[e] = now; break;
    case OP_ADMIT: {
      int victim, slot;
      const int rc = admit_warp(ls, hist_l, cfg, e, now, victim, slot);
      if (lane == 0) { io->rc = rc; io->out_i = victim; }
      break;
    }
    default: break;
  }
}

// ================================================================== host side

void init_layers(const DevCfg& cfg, int32_t init_fill, uint64_t seed, std::vector<LayerState>& out) {
  out.assign(cfg.L, LayerState{});
  const uint32_t E = cfg.E;
  const uint32_t c = std::min(cfg.slots, E);
  for (uint32_t l = 0; l < cfg.L; ++l) {
    LayerState& ls = out[l];
    std::memset(&ls, 0, sizeof ls);
    std::memset(ls.slot_of, -1, sizeof ls.slot_of);
    std::memset(ls.expert_of_slot, -1, sizeof ls.expert_of_slot);
    std::vector<uint32_t> res;
    if (init_fill == 0) {
      for (uint32_t i = 0; i < c; ++i) res.push_back(i);
    } else if (init_fill == 1) {
      // cache.cpp:26-39: seeded partial Fisher-Yates, sorted
      uint64_t rs[4];
      rng_seed(rs, derive_seed(seed, 0x11caffe0ULL + l));
      std::vector<uint32_t> pool(E);
      for (uint32_t i = 0; i < E; ++i) pool[i] = i;
      for (uint32_t i = 0; i < c; ++i) {
        const uint64_t j = i + rng_below(rs, E - i);
        std::swap(pool[i], pool[j]);
        res.push_back(pool[i]);
      }
      std::sort(res.begin(), res.end());
    }
    for (size_t i = 0; i < res.size(); ++i) {
      ls.mask |= 1ULL << res[i];
      ls.slot_of[res[i]] = (int8_t)i;
      ls.expert_of_slot[i] = (int8_t)res[i];
    }
    ls.n_res = (uint32_t)res.size();
  }
}

DevCfg make_dev_cfg(const moeb_config& c) {
  DevCfg d{};
  d.L = c.num_layers; d.E = c.experts; d.k = c.top_k; d.B = c.batch;
  d.alpha = c.alpha;
  d.slots = c.slots; d.window = c.window;
  d.policy = c.ce ? c.policy : 1;  // pipeline.cpp:64-70
  d.er = c.er; d.pre = c.pre; d.ba = c.ba;
  d.t_attn = c.t_attn; d.t_gpu = c.t_gpu; d.t_cpu_token = c.t_cpu_token; d.t_load = c.t_load;
  d.t_route = c.t_route;
  d.p_top = c.p_top; d.p_active = c.p_active;
  d.depth = c.queue_depth == 0 ? c.top_k : c.queue_depth;  // core.hpp:103-105
  return d;
}

// validate_config (core.cpp:30-70) violations, first one reported as
// simulate() does (pipeline.cpp:375-379), then the device-engine limits.
void validate(const moeb_config& c) {
  auto bad = [](const char* field, const char* rule) {
    throw Error(1, std::string("invalid config: ") + field + ": " + rule);
  };
  if (c.num_layers == 0) bad("shape.num_layers", "must be >= 1");
  if (c.experts == 0) bad("shape.experts_per_layer", "must be >= 1");
  if (c.top_k == 0) bad("shape.top_k", "must be >= 1");
  if (c.batch == 0) bad("shape.batch_size", "must be >= 1");
  if (c.top_k + 1 > c.experts) bad("shape.top_k", "k + 1 <= E required");
  if (!(c.alpha >= 0.0 && c.alpha < 1.0)) bad("router.alpha", "must satisfy 0 <= alpha < 1");
  if (c.slots > c.experts) bad("cache.slots_per_layer", "slots_per_layer <= E");
  if (c.window == 0) bad("cache.history_window", "must be >= 1");
  if (!(c.p_top >= 0.0 && c.p_top <= 1.0)) bad("predictor.p_top", "must be in [0, 1]");
  if (!(c.p_active >= 0.0 && c.p_active <= 1.0)) bad("predictor.p_active", "must be in [0, 1]");
  if (c.experts > (uint32_t)kMaxE) throw Error(1, "device engine: experts_per_layer must be <= 64");
  if (c.top_k > (uint32_t)kMaxK) throw Error(1, "device engine: top_k must be <= 16");
  if (c.batch > (uint32_t)kMaxB) throw Error(1, "device engine: batch_size must be <= 32");
}

static size_t replay_smem_bytes() { return sizeof(ReplaySmem); }

static void ensure_smem_attr() {
  static std::once_flag once;
  std::call_once(once, [] {
    MOEB_CUDA(cudaFuncSetAttribute(replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)replay_smem_bytes()));
    MOEB_CUDA(cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)replay_smem_bytes()));
  });
}

// --------------------------------------------------------------- result
struct Result {
  moeb_metrics m{};
  std::vector<moeb_task> tasks;
  std::vector<moeb_window> wins;
  std::vector<moeb_eviction> evs;
  std::vector<uint64_t> itc;
  std::vector<std::vector<uint32_t>> cache_final;
  std::vector<StepRec> steps;
  std::vector<TokRec> toks;
  uint32_t B = 0, E = 0;
  bool have_steps = false;
};

static void fill_metrics(moeb_metrics& m, const Counters& c, uint64_t iters, uint64_t total) {
  m = moeb_metrics{};
  m.demand_loads = c.demand; m.prefetch_loads = c.prefetch; m.cpu_computed = c.cpu_computed;
  m.hits = c.hits; m.misses = c.misses; m.substitutions = c.subs; m.low_score_kept = c.kept_low;
  m.selections = c.selections; m.iterations = iters; m.total_time = total;
  m.draws = c.draws; m.trace_supplied = c.trace_supplied; m.head_top = c.head_top;
  m.head_active = c.head_active; m.head_inactive = c.head_inactive; m.issued = c.issued;
  m.cancelled = c.cancelled;
  // pipeline.cpp:346-361
  m.tpot = iters == 0 ? 0.0 : (double)total / (double)iters;
  m.hit_rate = c.selections == 0 ? 0.0 : (double)c.hits / (double)c.selections;
  const uint64_t st = c.subs + c.kept_low;
  m.substitution_ratio = st == 0 ? 0.0 : (double)c.subs / (double)st;
}
void metrics_from_counters(moeb_metrics& m, const Counters& c, uint64_t iters, uint64_t total) {
  fill_metrics(m, c, iters, total);
}

static std::string list_json(const std::vector<uint32_t>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) s += ",";
    s += std::to_string(v[i]);
  }
  return s + "]";
}
static std::vector<uint32_t> mask_list(uint64_t m) {
  std::vector<uint32_t> v;
  for (uint32_t e = 0; e < 64; ++e)
    if ((m >> e) & 1ULL) v.push_back(e);
  return v;
}
static std::string num_json(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::string steps_json(const StepRec* steps, const TokRec* toks, size_t n, uint32_t B) {
  std::ostringstream j;
  j << "[";
  for (size_t i = 0; i < n; ++i) {
    const StepRec& r = steps[i];
    j << (i ? "," : "") << "{\"it\":" << r.it << ",\"layer\":" << r.layer
      << ",\"mask\":" << list_json(mask_list(r.mask_before)) << ",\"tok\":[";
    for (uint32_t t = 0; t < B; ++t) {
      const TokRec& tr = toks[i * B + t];
      std::vector<uint32_t> sel(tr.sel, tr.sel + tr.n_sel), kept(tr.kept, tr.kept + tr.n_kept);
      j << (t ? "," : "") << "{\"sel\":" << list_json(sel) << ",\"sub\":[";
      for (uint32_t s = 0; s < tr.n_sub; ++s)
        j << (s ? "," : "") << "[" << (int)tr.sub_d[s] << "," << (int)tr.sub_c[s] << "]";
      j << "],\"kept\":" << list_json(kept) << "}";
    }
    std::vector<uint32_t> ld(r.load, r.load + r.n_load), cp(r.cpu, r.cpu + r.n_cpu),
        pf(r.pref, r.pref + r.n_pref);
    j << "],\"load\":" << list_json(ld) << ",\"cpu\":" << list_json(cp) << ",\"pref\":" << list_json(pf)
      << ",\"evict\":[";
    for (uint32_t s = 0; s < r.n_evict; ++s)
      j << (s ? "," : "") << "[" << (int)r.ev_layer[s] << "," << (int)r.ev_e[s] << "]";
    j << "],\"completion\":" << r.completion << "}";
  }
  j << "]";
  return j.str();
}

static std::string result_json(const Result& r) {
  const moeb_metrics& m = r.m;
  std::ostringstream j;
  j << "{\"metrics\":{\"tpot\":" << num_json(m.tpot) << ",\"hit_rate\":" << num_json(m.hit_rate)
    << ",\"substitution_ratio\":" << num_json(m.substitution_ratio)
    << ",\"demand_loads\":" << m.demand_loads << ",\"prefetch_loads\":" << m.prefetch_loads
    << ",\"cpu_computed\":" << m.cpu_computed << ",\"hits\":" << m.hits << ",\"misses\":" << m.misses
    << ",\"substitutions\":" << m.substitutions << ",\"low_score_kept\":" << m.low_score_kept
    << ",\"selections\":" << m.selections << ",\"iterations\":" << m.iterations
    << ",\"total_time\":" << m.total_time << "},";
  j << "\"stats\":{\"draws\":" << m.draws << ",\"trace_supplied\":" << m.trace_supplied
    << ",\"head_top\":" << m.head_top << ",\"head_active\":" << m.head_active
    << ",\"head_inactive\":" << m.head_inactive << ",\"issued\":" << m.issued
    << ",\"cancelled\":" << m.cancelled << "},";
  j << "\"cache_final\":[";
  for (size_t l = 0; l < r.cache_final.size(); ++l) j << (l ? "," : "") << list_json(r.cache_final[l]);
  j << "],\"tasks\":[";
  for (size_t i = 0; i < r.tasks.size(); ++i) {
    const moeb_task& t = r.tasks[i];
    j << (i ? "," : "") << "[" << (int)t.resource << "," << (int)t.kind << "," << t.expert_layer << ","
      << t.expert << "," << t.start << "," << t.end << "," << t.layer << "," << t.iteration << "]";
  }
  j << "],\"windows\":[";
  for (size_t i = 0; i < r.wins.size(); ++i) {
    const moeb_window& w = r.wins[i];
    j << (i ? "," : "") << "[" << w.iteration << "," << w.layer << "," << w.attn_end << ","
      << w.route_end << "," << w.completion << "," << list_json(mask_list(w.selected)) << "]";
  }
  j << "],\"evictions\":[";
  for (size_t i = 0; i < r.evs.size(); ++i)
    j << (i ? "," : "") << "[" << r.evs[i].time << "," << r.evs[i].layer << "," << r.evs[i].expert << "]";
  j << "],\"iteration_completion\":[";
  for (size_t i = 0; i < r.itc.size(); ++i) j << (i ? "," : "") << r.itc[i];
  j << "]";
  if (r.have_steps) j << ",\"steps\":" << steps_json(r.steps.data(), r.toks.data(), r.steps.size(), r.B);
  j << "}";
  return j.str();
}

// Device engine run over a whole trace (simulate()).
static Result* run_simulate(const moeb_config& c, const double* scores, const double* pred,
                            const uint8_t* has_pred, uint64_t iters, bool record_steps) {
  validate(c);
  ensure_smem_attr();
  const DevCfg cfg = make_dev_cfg(c);
  const uint32_t L = cfg.L, E = cfg.E, B = cfg.B;
  std::vector<LayerState> layers;
  init_layers(cfg, c.init_fill, c.seed, layers);
  EngineState st{};
  rng_seed(st.rng, derive_seed(c.seed, 0x94ed1c70ULL));  // pipeline.cpp:62

  const size_t n_steps = (size_t)iters * L;
  const size_t elems = n_steps * B * E;
  DevBuf<double> d_scores(std::max<size_t>(elems, 1)), d_pred, d_hist((size_t)L * cfg.window * E);
  DevBuf<uint8_t> d_has;
  DevBuf<EngineState> d_st(1);
  DevBuf<LayerState> d_layers(L);
  cudaStream_t s = 0;
  if (elems) MOEB_CUDA(cudaMemcpy(d_scores.p, scores, elems * sizeof(double), cudaMemcpyHostToDevice));
  if (pred && has_pred && elems) {
    d_pred.alloc(elems);
    d_has.alloc(n_steps * B);
    MOEB_CUDA(cudaMemcpy(d_pred.p, pred, elems * sizeof(double), cudaMemcpyHostToDevice));
    MOEB_CUDA(cudaMemcpy(d_has.p, has_pred, n_steps * B, cudaMemcpyHostToDevice));
  }
  d_hist.zero(s);
  MOEB_CUDA(cudaMemcpy(d_st.p, &st, sizeof st, cudaMemcpyHostToDevice));
  MOEB_CUDA(cudaMemcpy(d_layers.p, layers.data(), L * sizeof(LayerState), cudaMemcpyHostToDevice));

  const uint32_t D = std::min<uint32_t>(E, B * cfg.k);
  const size_t cap_tasks = n_steps * (2 + 3 * (size_t)D + cfg.depth) + 16;
  const size_t cap_evs = n_steps * ((size_t)D + cfg.depth) + 16;
  DevBuf<TaskRec> d_tasks(cap_tasks);
  DevBuf<WinRec> d_wins(n_steps + 1);
  DevBuf<EvRec> d_evs(cap_evs);
  DevBuf<StepRec> d_steps;
  DevBuf<TokRec> d_toks;
  if (record_steps) {
    d_steps.alloc(n_steps + 1);
    d_toks.alloc((n_steps + 1) * B);
  }
  DevBuf<unsigned long long> d_counts(4);
  DevBuf<uint32_t> d_over(1);
  d_counts.zero(s);
  d_over.zero(s);

  ReplayArgs a{};
  a.cfg = cfg;
  a.st = d_st.p;
  a.layers = d_layers.p;
  a.hist = d_hist.p;
  a.scores = d_scores.p;
  a.pred = d_pred.p;
  a.has_pred = d_has.p;
  a.iters = iters;
  a.logs = Logs{d_tasks.p, d_wins.p, d_evs.p, d_steps.p, d_toks.p, d_counts.p,
                cap_tasks, n_steps + 1, cap_evs, record_steps ? n_steps + 1 : 0, d_over.p};
  a.record_steps = record_steps;
  replay_kernel<<<1, kThreads, replay_smem_bytes(), s>>>(a);
  MOEB_CUDA(cudaGetLastError());
  MOEB_CUDA(cudaDeviceSynchronize());

  MOEB_CUDA(cudaMemcpy(&st, d_st.p, sizeof st, cudaMemcpyDeviceToHost));
  if (st.err == 4) throw Error(4, "admit: expert already resident");
  if (st.err) throw Error(1, "classify: beta undefined, need at least k+1 experts");
  unsigned long long counts[4];
  uint32_t over = 0;
  MOEB_CUDA(cudaMemcpy(counts, d_counts.p, sizeof counts, cudaMemcpyDeviceToHost));
  MOEB_CUDA(cudaMemcpy(&over, d_over.p, sizeof over, cudaMemcpyDeviceToHost));
  if (over) throw Error(4, "device engine: log capacity exceeded");
  MOEB_CUDA(cudaMemcpy(layers.data(), d_layers.p, L * sizeof(LayerState), cudaMemcpyDeviceToHost));

  auto* r = new Result();
  r->B = B;
  r->E = E;
  r->tasks.resize(counts[0]);
  r->wins.resize(counts[1]);
  r->evs.resize(counts[2]);
  static_assert(sizeof(moeb_task) == sizeof(TaskRec), "layout");
  static_assert(sizeof(moeb_window) == sizeof(WinRec), "layout");
  static_assert(sizeof(moeb_eviction) == sizeof(EvRec), "layout");
  if (counts[0]) MOEB_CUDA(cudaMemcpy(r->tasks.data(), d_tasks.p, counts[0] * sizeof(TaskRec), cudaMemcpyDeviceToHost));
  if (counts[1]) MOEB_CUDA(cudaMemcpy(r->wins.data(), d_wins.p, counts[1] * sizeof(WinRec), cudaMemcpyDeviceToHost));
  if (counts[2]) MOEB_CUDA(cudaMemcpy(r->evs.data(), d_evs.p, counts[2] * sizeof(EvRec), cudaMemcpyDeviceToHost));
  // Timeline order (pipeline.cpp:362-368) refined to a total order.
  std::sort(r->tasks.begin(), r->tasks.end(), [](const moeb_task& x, const moeb_task& y) {
    return std::tie(x.start, x.resource, x.end, x.layer, x.iteration, x.kind, x.expert_layer, x.expert) <
           std::tie(y.start, y.resource, y.end, y.layer, y.iteration, y.kind, y.expert_layer, y.expert);
  });
  for (const moeb_window& w : r->wins)
    if (w.layer == L - 1) r->itc.push_back(w.completion);
  for (uint32_t l = 0; l < L; ++l) r->cache_final.push_back(mask_list(layers[l].mask));
  if (record_steps) {
    r->have_steps = true;
    r->steps.resize(n_steps);
    r->toks.resize(n_steps * B);
    if (n_steps) {
      MOEB_CUDA(cudaMemcpy(r->steps.data(), d_steps.p, n_steps * sizeof(StepRec), cudaMemcpyDeviceToHost));
      MOEB_CUDA(cudaMemcpy(r->toks.data(), d_toks.p, n_steps * B * sizeof(TokRec), cudaMemcpyDeviceToHost));
    }
  }
  fill_metrics(r->m, st.c, iters, st.now);
  return r;
}

// ---------------------------------------------------------- cache handle
struct Cache {
  DevCfg cfg{};
  DevBuf<LayerState> layers;
  DevBuf<double> hist;
  DevBuf<CacheIO> io;
  std::vector<LayerState> host;  // mirror refreshed on demand
};

static void cache_op(Cache* c, int32_t op, uint32_t layer, uint32_t e, uint64_t now, CacheIO* out) {
  if (layer >= c->cfg.L) throw Error(4, "cache: layer out of range");
  cache_op_kernel<<<1, 32>>>(c->cfg, c->layers.p, c->hist.p, op, layer, e, now, c->io.p);
  MOEB_CUDA(cudaGetLastError());
  if (out) MOEB_CUDA(cudaMemcpy(out, c->io.p, sizeof(CacheIO), cudaMemcpyDeviceToHost));
}

// ---------------------------------------------------------- route helper
static void run_route(const double* scores, uint32_t B, uint32_t E, const uint8_t* mask,
                      uint32_t k, double alpha, int mode, RouteIO& io) {
  if (E > (uint32_t)kMaxE) throw Error(1, "device engine: experts_per_layer must be <= 64");
  if (E <= k) throw Error(1, "classify: beta undefined, need at least k+1 experts");
  if (B > (uint32_t)kMaxB) throw Error(1, "device engine: batch_size must be <= 32");
  if (k > (uint32_t)kMaxK) throw Error(1, "device engine: top_k must be <= 16");
  ensure_smem_attr();
  uint64_t m = 0;
  for (uint32_t e = 0; e < E; ++e)
    if (mask && mask[e]) m |= 1ULL << e;
  DevBuf<double> d_s(std::max<size_t>((size_t)B * E, 1));
  DevBuf<RouteIO> d_io(1);
  if (B) MOEB_CUDA(cudaMemcpy(d_s.p, scores, (size_t)B * E * sizeof(double), cudaMemcpyHostToDevice));
  MOEB_CUDA(cudaMemcpy(d_io.p, &io, sizeof io, cudaMemcpyHostToDevice));
  route_kernel<<<1, kThreads, replay_smem_bytes()>>>(d_s.p, B, E, m, k, alpha, mode, d_io.p);
  MOEB_CUDA(cudaGetLastError());
  MOEB_CUDA(cudaMemcpy(&io, d_io.p, sizeof io, cudaMemcpyDeviceToHost));
}

static void export_route(const RouteIO& io, uint32_t B, uint32_t k, uint32_t* sel, uint32_t* n_sel,
                         uint32_t* sub, uint32_t* n_sub, uint32_t* kept, uint32_t* n_kept,
                         uint32_t* top_set, uint32_t* n_top_set, uint32_t* pending,
                         uint32_t* n_pending) {
  for (uint32_t t = 0; t < B; ++t) {
    if (n_sel) n_sel[t] = io.nsel[t];
    if (n_sub) n_sub[t] = io.nsub[t];
    if (n_kept) n_kept[t] = io.nkept[t];
    for (uint32_t i = 0; i < k; ++i) {
      if (sel) sel[t * k + i] = i < io.nsel[t] ? io.sel[t][i] : 0;
      if (kept) kept[t * k + i] = i < io.nkept[t] ? io.kept[t][i] : 0;
      if (sub) {
        sub[(t * k + i) * 2] = i < io.nsub[t] ? io.sub_d[t][i] : 0;
        sub[(t * k + i) * 2 + 1] = i < io.nsub[t] ? io.sub_c[t][i] : 0;
      }
    }
  }
  if (top_set) {
    uint32_t n = 0;
    for (uint32_t e : mask_list(io.C)) top_set[n++] = e;
    if (n_top_set) *n_top_set = n;
  }
  if (pending) {
    uint32_t n = 0;
    for (uint32_t e : mask_list(io.pending)) pending[n++] = e;
    if (n_pending) *n_pending = n;
  }
}

}  // namespace moeb

using namespace moeb;

// ==================================================================== C-ABI
extern "C" {

const char* moeb_last_error(void) { return g_last_error.c_str(); }

int moeb_device_count(int* n) {
  return guarded([&] { MOEB_CUDA(cudaGetDeviceCount(n)); });
}

void moeb_free(void* p) { std::free(p); }

int moeb_classify(const double* scores, uint32_t E, uint32_t k, double alpha, double* thr,
                  uint32_t* actives, uint32_t* top, uint32_t* n_top, uint32_t* low, uint32_t* n_low,
                  uint32_t* alt, uint32_t* n_alt) {
  return guarded([&] {
    RouteIO io{};
    run_route(scores, 1, E, nullptr, k, alpha, 3, io);
    for (int i = 0; i < 4; ++i) thr[i] = io.thr[i];
    uint32_t nt = 0, nl = 0, na = 0;
    for (uint32_t r = 0; r < E; ++r) {
      const uint32_t e = io.order[r];
      if (r < k) {
        if (actives) actives[r] = e;
        if ((io.top >> e) & 1ULL) top[nt++] = e;
        if ((io.low >> e) & 1ULL) low[nl++] = e;
      } else if ((io.alt >> e) & 1ULL) {
        alt[na++] = e;
      }
    }
    *n_top = nt;
    *n_low = nl;
    *n_alt = na;
  });
}

int moeb_plain_top_k(const double* scores, uint32_t E, uint32_t k, uint32_t* out, uint32_t* n_out) {
  return guarded([&] {
    const uint32_t n = std::min(k, E);
    if (n == 0) { *n_out = 0; return; }
    if (E > (uint32_t)kMaxE) throw Error(1, "device engine: experts_per_layer must be <= 64");
    RouteIO io{};
    // ranking needs k < E for classify's beta; plain_top_k has no such rule,
    // so rank with k' = 0 and take the prefix of the full order.
    run_route(scores, 1, E, nullptr, 0, 0.0, 4, io);
    for (uint32_t i = 0; i < n; ++i) out[i] = io.order[i];
    *n_out = n;
  });
}

int moeb_route(const double* scores, uint32_t B, uint32_t E, const uint8_t* resident_mask,
               uint32_t k, double alpha, int32_t coalesce, uint32_t* sel, uint32_t* n_sel,
               uint32_t* sub, uint32_t* n_sub, uint32_t* kept, uint32_t* n_kept,
               uint32_t* top_set, uint32_t* n_top_set, uint32_t* pending, uint32_t* n_pending) {
  return guarded([&] {
    RouteIO io{};
    run_route(scores, B, E, resident_mask, k, alpha, coalesce ? 1 : 0, io);
    export_route(io, B, k, sel, n_sel, sub, n_sub, kept, n_kept, top_set, n_top_set, pending, n_pending);
  });
}

int moeb_coalesce(const double* scores, uint32_t B, uint32_t E, const uint8_t* resident_mask,
                  uint32_t k, const double* thresholds, uint32_t* sel, uint32_t* n_sel, uint32_t* sub,
                  uint32_t* n_sub, uint32_t* kept, uint32_t* n_kept, const uint32_t* top_set,
                  uint32_t n_top_set, uint32_t* pending, uint32_t* n_pending) {
  return guarded([&] {
    if (B > (uint32_t)kMaxB) throw Error(1, "device engine: batch_size must be <= 32");
    RouteIO io{};
    for (uint32_t t = 0; t < B; ++t) {
      io.nsel[t] = (uint8_t)n_sel[t];
      io.nsub[t] = (uint8_t)n_sub[t];
      io.nkept[t] = (uint8_t)n_kept[t];
      for (uint32_t i = 0; i < k && i < (uint32_t)kMaxK; ++i) {
        io.sel[t][i] = (uint8_t)sel[t * k + i];
        io.kept[t][i] = (uint8_t)kept[t * k + i];
        io.sub_d[t][i] = (uint8_t)sub[(t * k + i) * 2];
        io.sub_c[t][i] = (uint8_t)sub[(t * k + i) * 2 + 1];
      }
    }
    for (uint32_t i = 0; i < n_top_set; ++i) io.C |= 1ULL << top_set[i];
    for (uint32_t t = 0; t < B; ++t)
      for (int j = 0; j < 4; ++j) io.thr_tok[t][j] = thresholds[t * 4 + j];
    if (B == 0) { *n_pending = 0; return; }
    run_route(scores, B, E, resident_mask, k, 0.0, 2, io);
    export_route(io, B, k, sel, n_sel, sub, n_sub, kept, n_kept, nullptr, nullptr, pending, n_pending);
  });
}

int moeb_balance(const uint32_t* uid, const uint32_t* batch, uint32_t n, uint64_t t_cpu_token,
                 uint64_t t_load, uint32_t* load_list, uint32_t* n_load, uint32_t* cpu_list,
                 uint32_t* n_cpu, uint64_t* c_load, uint64_t* c_cpu) {
  return guarded([&] {
    if (n > (uint32_t)kMaxE) throw Error(1, "device engine: at most 64 demand items");
    // the device kernel carries 8-bit uids; remap arbitrary uids by rank
    std::vector<uint32_t> uids(uid, uid + n);
    std::vector<uint32_t> sorted = uids;
    std::sort(sorted.begin(), sorted.end());
    BalanceIO io{};
    io.n = n;
    for (uint32_t i = 0; i < n; ++i) {
      io.uid[i] = (uint8_t)(std::lower_bound(sorted.begin(), sorted.end(), uids[i]) - sorted.begin());
      if (batch[i] > 0xffff) throw Error(1, "device engine: batch exceeds 65535");
      io.batch[i] = (uint16_t)batch[i];
    }
    DevBuf<BalanceIO> d(1);
    MOEB_CUDA(cudaMemcpy(d.p, &io, sizeof io, cudaMemcpyHostToDevice));
    balance_kernel<<<1, 32>>>(d.p, t_cpu_token, t_load);
    MOEB_CUDA(cudaGetLastError());
    MOEB_CUDA(cudaMemcpy(&io, d.p, sizeof io, cudaMemcpyDeviceToHost));
    uint64_t cl = 0, cc = 0;
    std::vector<uint32_t> bat_of(n);
    for (uint32_t i = 0; i < n; ++i) bat_of[io.uid[i]] = batch[i];
    for (uint32_t i = 0; i < io.n_load; ++i) { load_list[i] = sorted[io.load[i]]; cl += t_load; }
    for (uint32_t i = 0; i < io.n_cpu; ++i) {
      cpu_list[i] = sorted[io.cpu[i]];
      cc += (uint64_t)bat_of[io.cpu[i]] * t_cpu_token;
    }
    *n_load = io.n_load;
    *n_cpu = io.n_cpu;
    if (c_load) *c_load = cl;
    if (c_cpu) *c_cpu = cc;
  });
}

int moeb_predict_scores(const double* true_next, const double* supplied, uint32_t E, double p_top,
                        double p_active, uint32_t k, double alpha, uint64_t* rng_state, double* out,
                        uint32_t* head, int32_t* head_kind) {
  return guarded([&] {
    if (E > (uint32_t)kMaxE) throw Error(1, "device engine: experts_per_layer must be <= 64");
    if (E <= k) throw Error(1, "classify: beta undefined, need at least k+1 experts");
    PredictIO io{};
    std::memcpy(io.tn, true_next, E * sizeof(double));
    if (supplied) std::memcpy(io.sup, supplied, E * sizeof(double));
    io.supplied = supplied != nullptr;
    std::memcpy(io.rng, rng_state, sizeof io.rng);
    DevBuf<PredictIO> d(1);
    MOEB_CUDA(cudaMemcpy(d.p, &io, sizeof io, cudaMemcpyHostToDevice));
    predict_kernel<<<1, 32>>>(d.p, E, k, alpha, p_top, p_active);
    MOEB_CUDA(cudaGetLastError());
    MOEB_CUDA(cudaMemcpy(&io, d.p, sizeof io, cudaMemcpyDeviceToHost));
    std::memcpy(out, io.out, E * sizeof(double));
    std::memcpy(rng_state, io.rng, sizeof io.rng);
    *head = io.head;
    *head_kind = io.kind;
  });
}

int moeb_build_queue(const double* predicted, const uint8_t* resident_mask, uint32_t E,
                     uint32_t depth, uint32_t* entries, uint32_t* n_entries) {
  return guarded([&] {
    if (E > (uint32_t)kMaxE) throw Error(1, "device engine: experts_per_layer must be <= 64");
    *n_entries = 0;
    if (depth == 0 || E == 0) return;  // prefetch.cpp:92-94
    QueueIO io{};
    std::memcpy(io.pred, predicted, E * sizeof(double));
    for (uint32_t e = 0; e < E; ++e)
      if (resident_mask[e]) io.mask |= 1ULL << e;
    DevBuf<QueueIO> d(1);
    MOEB_CUDA(cudaMemcpy(d.p, &io, sizeof io, cudaMemcpyHostToDevice));
    queue_kernel<<<1, 32>>>(d.p, E, depth);
    MOEB_CUDA(cudaGetLastError());
    MOEB_CUDA(cudaMemcpy(&io, d.p, sizeof io, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < io.n; ++i) entries[i] = io.ent[i];
    *n_entries = io.n;
  });
}

// ---- cache
struct moeb_cache : moeb::Cache {};

int moeb_cache_create(uint32_t layers, uint32_t E, uint32_t slots, uint32_t window, int32_t policy,
                      int32_t init_fill, uint64_t seed, moeb_cache** out) {
  return guarded([&] {
    if (E > (uint32_t)kMaxE) throw Error(1, "device engine: experts_per_layer must be <= 64");
    auto* c = new moeb_cache();
    c->cfg.L = layers;
    c->cfg.E = E;
    c->cfg.slots = slots;
    c->cfg.window = window;
    c->cfg.policy = policy;
    std::vector<LayerState> ls;
    init_layers(c->cfg, init_fill, seed, ls);
    c->layers.alloc(std::max<uint32_t>(layers, 1));
    c->hist.alloc(std::max<size_t>((size_t)layers * window * E, 1));
    c->hist.zero();
    c->io.alloc(1);
    if (layers) MOEB_CUDA(cudaMemcpy(c->layers.p, ls.data(), layers * sizeof(LayerState), cudaMemcpyHostToDevice));
    *out = c;
  });
}

void moeb_cache_destroy(moeb_cache* c) { delete c; }

int moeb_cache_resident(moeb_cache* c, uint32_t layer, uint32_t* out, uint32_t* n) {
  return guarded([&] {
    if (layer >= c->cfg.L) throw Error(4, "cache: layer out of range");
    LayerState ls;
    MOEB_CUDA(cudaMemcpy(&ls, c->layers.p + layer, sizeof ls, cudaMemcpyDeviceToHost));
    uint32_t i = 0;
    for (uint32_t e : mask_list(ls.mask)) out[i++] = e;
    *n = i;
  });
}

int moeb_cache_record(moeb_cache* c, uint32_t layer, const double* scores, uint32_t n) {
  return guarded([&] {
    if (n != c->cfg.E) throw Error(4, "record_scores: score vector length mismatch");
    CacheIO io{};
    std::memcpy(io.v, scores, n * sizeof(double));
    MOEB_CUDA(cudaMemcpy(c->io.p, &io, sizeof io, cudaMemcpyHostToDevice));
    cache_op(c, OP_RECORD, layer, 0, 0, nullptr);
  });
}

int moeb_cache_window_average(moeb_cache* c, uint32_t layer, uint32_t e, double* out) {
  return guarded([&] {
    CacheIO io{};
    cache_op(c, OP_AVG, layer, e, 0, &io);
    *out = io.out_d;
  });
}

int moeb_cache_try_evict(moeb_cache* c, uint32_t layer, int64_t* victim) {
  return guarded([&] {
    CacheIO io{};
    cache_op(c, OP_EVICT, layer, 0, 0, &io);
    *victim = io.out_i;
  });
}

int moeb_cache_shield(moeb_cache* c, uint32_t layer, uint32_t e) {
  return guarded([&] { cache_op(c, OP_SHIELD, layer, e, 0, nullptr); });
}

int moeb_cache_unshield_layer(moeb_cache* c, uint32_t layer) {
  return guarded([&] { cache_op(c, OP_UNSHIELD, layer, 0, 0, nullptr); });
}

int moeb_cache_is_shielded(moeb_cache* c, uint32_t layer, uint32_t e, int32_t* out) {
  return guarded([&] {
    if (layer >= c->cfg.L) throw Error(4, "cache: layer out of range");
    LayerState ls;
    MOEB_CUDA(cudaMemcpy(&ls, c->layers.p + layer, sizeof ls, cudaMemcpyDeviceToHost));
    *out = (int32_t)((ls.shield >> e) & 1ULL);
  });
}

int moeb_cache_touch(moeb_cache* c, uint32_t layer, uint32_t e, uint64_t now) {
  return guarded([&] { cache_op(c, OP_TOUCH, layer, e, now, nullptr); });
}

int moeb_cache_admit(moeb_cache* c, uint32_t layer, uint32_t e, uint64_t now, int64_t* evicted) {
  return guarded([&] {
    CacheIO io{};
    cache_op(c, OP_ADMIT, layer, e, now, &io);
    if (evicted) *evicted = io.out_i;
    if (io.rc == 3) throw Error(3, "no evictable expert");
    if (io.rc == 4) throw Error(4, "admit: expert already resident");
  });
}

// ---- simulate
struct moeb_result : moeb::Result {};

int moeb_simulate(const moeb_config* cfg, const double* scores, const double* pred,
                  const uint8_t* has_pred, uint64_t iters, int32_t record_steps, moeb_result** out) {
  return guarded([&] {
    Result* r = run_simulate(*cfg, scores, pred, has_pred, iters, record_steps != 0);
    auto* rr = new moeb_result();
    static_cast<Result&>(*rr) = std::move(*r);
    delete r;
    *out = rr;
  });
}

int moeb_result_json(const moeb_result* r, char** json) {
  return guarded([&] {
    const std::string s = result_json(*r);
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    *json = p;
  });
}

int moeb_result_metrics(const moeb_result* r, moeb_metrics* m) {
  *m = r->m;
  return 0;
}
int moeb_result_tasks(const moeb_result* r, const moeb_task** tasks, size_t* n) {
  *tasks = r->tasks.data();
  *n = r->tasks.size();
  return 0;
}
int moeb_result_windows(const moeb_result* r, const moeb_window** w, size_t* n) {
  *w = r->wins.data();
  *n = r->wins.size();
  return 0;
}
int moeb_result_evictions(const moeb_result* r, const moeb_eviction** ev, size_t* n) {
  *ev = r->evs.data();
  *n = r->evs.size();
  return 0;
}
int moeb_result_iteration_completion(const moeb_result* r, const uint64_t** t, size_t* n) {
  *t = r->itc.data();
  *n = r->itc.size();
  return 0;
}
int moeb_result_cache_final(const moeb_result* r, uint32_t layer, uint32_t* out, uint32_t* n) {
  if (layer >= r->cache_final.size()) return 4;
  const auto& v = r->cache_final[layer];
  for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
  *n = (uint32_t)v.size();
  return 0;
}
void moeb_result_free(moeb_result* r) { delete r; }

}  // extern "C"
