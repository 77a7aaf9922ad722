// decide.cuh — one (iteration, layer) decision step on the device.
//
// decide_step() restates Simulator::run_layer (pipeline.cpp:128-286) and
// Simulator::schedule_prefetch (pipeline.cpp:293-344) with the policies they
// call: route (router.cpp:97-152), coalesce_for_batching (router.cpp:154-260),
// plain_top_k (router.cpp:35-39), CacheState (cache.cpp:58-156), balance
// (balancer.cpp:8-38), predict_scores / build_queue (prefetch.cpp:34-115).
// Called by the whole decision CTA (kThreads threads).
#pragma once

#include "engine.cuh"

namespace moeb {

// Pointers may be global or shared (callers stage hot state in smem). When
// the prefetch target is the executing layer (L == 1), tls == ls and
// thist == hist_l.
struct StepCtx {
  const DevCfg* cfg;
  EngineState* st;
  LayerState* ls;        // executing layer
  double* hist_l;        // its score ring [window][E]
  LayerState* tls;       // prefetch target layer
  double* thist;         // its score ring
  const Logs* logs;      // nullable
  uint64_t it;
  uint32_t layer;
  uint32_t has_target;   // prefetch target exists (pipeline.cpp:401-409)
  uint32_t target_layer;
  uint64_t target_it;
  uint64_t* prof;        // nullable: phase timers (globaltimer deltas)
  // predictor mode (the partial-forward predictor): the
  // step leaves its schedule_prefetch pending (the prediction for the next
  // layer needs this layer's FFN), and the next step runs it first
  // (run_pending), with every token's prediction supplied in sm->np.
  uint32_t defer_prefetch;
  uint32_t run_pending;
  StepRec* prev_rec;     // nullable: the previous step's record (gets the pending phase's issues)
  uint32_t f32_scores;   // every score is an fp32 value (the stack): integer-key ranking
};

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Phase timers of the decision CTA (make PROFILE=1): the SM cycle counter
// (cycle resolution; %globaltimer ticks far more coarsely), in ns at the
// B200's 1965 MHz boost clock the bench runs at.
__device__ __forceinline__ uint64_t ptimer() { return (uint64_t)clock64() * 1000ull / 1965ull; }

// Extra shared state for the prefetch target's classification.
struct NextSmem {
  uint8_t order[kMaxB][kMaxE];
  uint64_t act[kMaxB], top[kMaxB];
};

// ------------------------------------------------------- cache helpers
// cache.cpp:69-79: sum oldest -> newest, then divide by the window size.
__device__ __forceinline__ double window_average(const LayerState* ls, const double* hist_l,
                                                 uint32_t window, uint32_t E, uint32_t e) {
  if (ls->h_size == 0) return 0.0;
  double sum = 0.0;
  uint32_t slot = ls->h_head;
  for (uint32_t i = 0; i < ls->h_size; ++i) {
    sum += hist_l[(size_t)slot * E + e];
    slot = (slot + 1 == window) ? 0 : slot + 1;
  }
  return sum / (double)ls->h_size;
}

// cache.cpp:81-106 (warp-collective; every lane returns the victim or -1).
// avg: optional precomputed window averages of this layer (the history does
// not change between a step's record_scores and its admissions).
__device__ inline int try_evict_warp(const LayerState* ls, const double* hist_l, const DevCfg& cfg,
                                     const double* avg = nullptr) {
  const int lane = lane_id();
  const uint64_t cand = ls->mask & ~ls->shield;
  if (cfg.policy == 0) {
    double key = 0.0;
    uint32_t idx = 0xffffffffu;
    for (uint32_t e = lane; e < cfg.E; e += 32) {
      if (!has(cand, e)) continue;
      const double a = avg ? avg[e] : window_average(ls, hist_l, cfg.window, cfg.E, e);
      if (idx == 0xffffffffu || a < key) { key = a; idx = e; }
    }
    warp_argmin_d(key, idx);
    return idx == 0xffffffffu ? -1 : (int)idx;
  }
  uint64_t key = 0;
  uint32_t idx = 0xffffffffu;
  for (uint32_t e = lane; e < cfg.E; e += 32) {
    if (!has(cand, e)) continue;
    const uint64_t a = ls->last_access[e];
    if (idx == 0xffffffffu || a < key) { key = a; idx = e; }
  }
  warp_argmin_u(key, idx);
  return idx == 0xffffffffu ? -1 : (int)idx;
}

// cache.cpp:136-156. Returns 0 ok, 3 CacheError (all shielded), 4 already
// resident. victim/slot are -1 when none. Warp-collective.
__device__ inline int admit_warp(LayerState* ls, const double* hist_l, const DevCfg& cfg,
                                 uint32_t e, uint64_t now, int& victim, int& slot,
                                 const double* avg = nullptr) {
  const int lane = lane_id();
  victim = -1;
  slot = -1;
  if (has(ls->mask, e)) return 4;
  if (cfg.slots == 0) return 0;  // zero-slot cache: loads pass through
  if (ls->n_res >= cfg.slots) {
    const int v = try_evict_warp(ls, hist_l, cfg, avg);
    if (v < 0) return 3;
    victim = v;
    slot = ls->slot_of[v];
    __syncwarp();
    if (lane == 0) {
      ls->mask &= ~bit(v);
      ls->n_res -= 1;
      ls->slot_of[v] = -1;
      if (slot >= 0) ls->expert_of_slot[slot] = -1;
    }
    __syncwarp();
  }
  if (slot < 0) {
    const uint32_t nslot = cfg.slots < (uint32_t)kMaxSlots ? cfg.slots : (uint32_t)kMaxSlots;
    const bool f0 = (uint32_t)lane < nslot && ls->expert_of_slot[lane] < 0;
    const bool f1 = (uint32_t)lane + 32 < nslot && ls->expert_of_slot[lane + 32] < 0;
    const uint64_t free_mask = ballot64(f0, f1);
    slot = free_mask ? __ffsll((long long)free_mask) - 1 : -1;
  }
  __syncwarp();
  if (lane == 0) {
    ls->mask |= bit(e);
    ls->n_res += 1;
    ls->last_access[e] = now;
    ls->slot_of[e] = (int8_t)slot;
    if (slot >= 0) ls->expert_of_slot[slot] = (int8_t)e;
  }
  __syncwarp();
  return 0;
}

// cache.cpp:58-67: push one score vector into the ring (warp-collective).
__device__ inline void record_scores_warp(LayerState* ls, double* hist_l, uint32_t window,
                                          uint32_t E, const double* v) {
  uint32_t slot;
  const uint32_t head = ls->h_head, size = ls->h_size;
  if (size < window) {
    slot = head + size;
    if (slot >= window) slot -= window;
  } else {
    slot = head;
  }
  for (uint32_t e = lane_id(); e < E; e += 32) hist_l[(size_t)slot * E + e] = v[e];
  __syncwarp();
  if (lane_id() == 0) {
    if (size < window) {
      ls->h_size = size + 1;
    } else {
      ls->h_head = (head + 1 == window) ? 0 : head + 1;
    }
  }
  __syncwarp();
}

// Warp-wide: lane t < B holds token t's selection mask; cnt[e] = number of
// tokens selecting e (masks exchanged through shared memory: B reads per lane).
__device__ inline void batch_counts(uint64_t m, uint32_t B, uint32_t E, uint16_t* cnt) {
  __shared__ uint64_t s_selm[kMaxB];
  const uint32_t lane = lane_id();
  __syncwarp();
  if (lane < B) s_selm[lane] = m;
  __syncwarp();
  for (uint32_t e = lane; e < E; e += 32) {
    uint32_t c = 0;
    for (uint32_t t = 0; t < B; ++t) c += (uint32_t)(s_selm[t] >> e) & 1u;
    cnt[e] = (uint16_t)c;
  }
  __syncwarp();
}

// --------------------------------------------------------- router parts
// router.cpp:114-149: pass 2 for token t (executed by one lane).
__device__ inline void route_token(DecideSmem* sm, uint32_t t, uint64_t resident, uint32_t E,
                                   uint32_t k) {
  const uint64_t free_set = resident | sm->C;
  const uint8_t* order = sm->order[t];
  const uint64_t top = sm->top[t], low = sm->low[t], alt = sm->alt[t];
  uint32_t n = 0, nk = 0, ns = 0;
  for (uint32_t r = 0; r < k; ++r) {
    const uint32_t e = order[r];
    if (has(top, e)) sm->sel[t][n++] = (uint8_t)e;
  }
  uint8_t blow[kMaxK];
  uint32_t m = 0;
  for (uint32_t r = 0; r < k; ++r) {
    const uint32_t e = order[r];
    if (!has(low, e)) continue;
    if (has(free_set, e)) sm->sel[t][n++] = (uint8_t)e;
    else blow[m++] = (uint8_t)e;
  }
  uint8_t alts[kMaxK];
  uint32_t na = 0;
  for (uint32_t r = k; r < E && na < m; ++r) {
    const uint32_t e = order[r];
    if (has(alt, e) && has(free_set, e)) alts[na++] = (uint8_t)e;
  }
  const uint32_t covered = m < na ? m : na;
  const uint32_t kept = m - covered;
  for (uint32_t i = 0; i < kept; ++i) {
    sm->sel[t][n++] = blow[i];
    sm->kept[t][nk++] = blow[i];
  }
  for (uint32_t i = 0; i < covered; ++i) {
    sm->sel[t][n++] = alts[i];
    sm->sub_d[t][ns] = blow[kept + i];
    sm->sub_c[t][ns] = alts[i];
    ++ns;
  }
  sm->nsel[t] = (uint8_t)n;
  sm->nkept[t] = (uint8_t)nk;
  sm->nsub[t] = (uint8_t)ns;
}

// The same pass 2 for token t, bit-parallel on one warp: lane l handles
// ranks l and l + 32. Every list of the reference is in rank order, so the
// rank-space masks (bit r = the expert at rank r is in the set) give each
// entry's output position by a popcount of the lower ranks — no serial scan.
__device__ __forceinline__ uint32_t popc_below(uint64_t m, uint32_t r) {
  return (uint32_t)__popcll(m & ((1ULL << r) - 1ULL));
}
__device__ inline void route_token_warp(DecideSmem* sm, uint32_t t, uint64_t resident, uint32_t E,
                                        uint32_t k, uint64_t C) {
  const uint32_t lane = (uint32_t)lane_id();
  const uint64_t free_set = resident | C;
  const uint8_t* order = sm->order[t];
  const uint64_t top = sm->top[t], low = sm->low[t], alt = sm->alt[t];
  const uint32_t r0 = lane, r1 = lane + 32;
  const bool v0 = r0 < E, v1 = r1 < E;
  const uint32_t x0 = v0 ? order[r0] : 0u, x1 = v1 ? order[r1] : 0u;
  const bool a0 = v0 && r0 < k, a1 = v1 && r1 < k;  // active ranks
  const uint64_t top_r = ballot64(a0 && has(top, x0), a1 && has(top, x1));
  const uint64_t lowfree_r = ballot64(a0 && has(low, x0) && has(free_set, x0), a1 && has(low, x1) && has(free_set, x1));
  const uint64_t blow_r = ballot64(a0 && has(low, x0) && !has(free_set, x0), a1 && has(low, x1) && !has(free_set, x1));
  const uint64_t alt_r = ballot64(v0 && !a0 && has(alt, x0) && has(free_set, x0),
                                  v1 && !a1 && has(alt, x1) && has(free_set, x1));
  const uint32_t nt = __popcll(top_r), nf = __popcll(lowfree_r), m = __popcll(blow_r);
  const uint32_t na = __popcll(alt_r);
  const uint32_t covered = m < na ? m : na;
  const uint32_t kept = m - covered;
  auto place = [&](uint32_t r, uint32_t x) {
    const uint64_t b = 1ULL << r;
    if (top_r & b) {
      sm->sel[t][popc_below(top_r, r)] = (uint8_t)x;
    } else if (lowfree_r & b) {
      sm->sel[t][nt + popc_below(lowfree_r, r)] = (uint8_t)x;
    } else if (blow_r & b) {
      const uint32_t j = popc_below(blow_r, r);
      if (j < kept) {  // the strongest uncovered lows are kept
        sm->sel[t][nt + nf + j] = (uint8_t)x;
        sm->kept[t][j] = (uint8_t)x;
      } else {         // the weakest are replaced, pairwise with the alternatives
        sm->sub_d[t][j - kept] = (uint8_t)x;
      }
    } else if (alt_r & b) {
      const uint32_t j = popc_below(alt_r, r);
      if (j < covered) {
        sm->sel[t][nt + nf + kept + j] = (uint8_t)x;
        sm->sub_c[t][j] = (uint8_t)x;
      }
    }
  };
  if (v0) place(r0, x0);
  if (v1) place(r1, x1);
  if (lane == 0) {
    sm->nsel[t] = (uint8_t)(nt + nf + m);
    sm->nkept[t] = (uint8_t)kept;
    sm->nsub[t] = (uint8_t)covered;
  }
  __syncwarp();
}

// Order-preserving unsigned key of a double (-0.0 folded onto +0.0, as the
// reference's `>` treats them equal).
__device__ __forceinline__ uint64_t dkey(double v) {
  if (v == 0.0) v = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

// router.cpp:154-248: fixed-point coalescing, warp 0. The reference scans
// candidates x ascending and replaces the best on more others, or equal
// others and a higher score: the winner is the lexicographic max of
// (others, score, -x) over the candidates whose count beats the occupant's.
// Each lane evaluates experts lane and lane + 32 (the lower one wins its
// local ties), then four warp reductions (redux.sync) find the winner:
// max count, max score (hi then lo word of the order-preserving key), min x.
// The band of every token (beta > 0, R <= s < L) is a bitmask computed once.
__device__ inline void coalesce_warp(DecideSmem* sm, uint32_t B, uint32_t E, uint32_t k,
                                     uint64_t resident, uint16_t* cnt) {
  const uint32_t lane = (uint32_t)lane_id();
  // batch counts: a token's selection is a set, so cnt[e] = number of
  // tokens (lanes, B <= 32) whose selection mask holds e
  {
    uint64_t m = 0;
    if (lane < B)
      for (uint32_t i = 0; i < sm->nsel[lane]; ++i) m |= bit(sm->sel[lane][i]);
    batch_counts(m, B, E, cnt);
  }
  __shared__ uint64_t s_band[kMaxB];
  for (uint32_t t = 0; t < B; ++t) {
    const double* s = sm->s[t];
    const double beta = sm->beta[t], thR = sm->thR[t], thL = sm->thL[t];
    const bool b0 = lane < E && beta > 0.0 && s[lane] >= thR && s[lane] < thL;
    const bool b1 = lane + 32 < E && beta > 0.0 && s[lane + 32] >= thR && s[lane + 32] < thL;
    const uint64_t bm = ballot64(b0, b1) & ~sm->act[t];
    if (lane == 0) s_band[t] = bm;
  }
  __syncwarp();
  const uint64_t avail = resident | sm->C;
  bool changed = true;
  while (changed) {
    changed = false;
    for (uint32_t t = 0; t < B; ++t) {
      const uint64_t low = sm->low[t];
      if (!low) continue;
      const double* s = sm->s[t];
      const uint64_t band = s_band[t];
      // the token's selection as a mask: lane i holds entry i (k <= 16 < 32)
      uint64_t selm;
      {
        const uint32_t e = lane < sm->nsel[t] ? sm->sel[t][lane] : 64u;
        const uint32_t lo = __reduce_or_sync(0xffffffffu, e < 32 ? 1u << e : 0u);
        const uint32_t hi = __reduce_or_sync(0xffffffffu, (e >= 32 && e < 64) ? 1u << (e - 32) : 0u);
        selm = (uint64_t)lo | ((uint64_t)hi << 32);
      }
      for (uint32_t r = 0; r < k; ++r) {
        const uint32_t orig = sm->order[t][r];
        if (!has(low, orig)) continue;
        // the slot's occupant: a kept low is its own; a substituted one, its
        // substitute (lane i checks list entry i: first match as the scans)
        const uint32_t km = __ballot_sync(0xffffffffu, lane < sm->nkept[t] && sm->kept[t][lane] == orig);
        const uint32_t smk = __ballot_sync(0xffffffffu, lane < sm->nsub[t] && sm->sub_d[t][lane] == orig);
        const int kept_pos = km ? __ffs(km) - 1 : -1;
        int sub_pos = -1;
        uint32_t occupant;
        if (kept_pos >= 0) {
          occupant = orig;
        } else {
          if (!smk) continue;
          sub_pos = __ffs(smk) - 1;
          occupant = sm->sub_c[t][sub_pos];
        }
        const uint32_t occ_others = cnt[occupant] - 1u;
        const uint64_t cand = band & ~selm;
        // local best of the lane's two experts (x0 < x1: x0 wins ties)
        uint32_t bc = 0, bx = 0xffffffffu;  // bc = others + 1 (0: none)
        uint64_t bk = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t x = lane + 32u * h;
          if (x >= E || !has(cand, x)) continue;
          const uint32_t others = cnt[x];
          if (!(has(avail, x) || others > 0) || others <= occ_others) continue;
          const uint64_t key = dkey(s[x]);
          if (bx == 0xffffffffu || others + 1 > bc || (others + 1 == bc && key > bk)) {
            bc = others + 1;
            bk = key;
            bx = x;
          }
        }
        const uint32_t mc = __reduce_max_sync(0xffffffffu, bc);
        if (mc == 0) continue;  // best == occupant
        const bool m1 = bc == mc;
        const uint32_t hi = m1 ? (uint32_t)(bk >> 32) : 0u;
        const uint32_t mhi = __reduce_max_sync(0xffffffffu, hi);
        const bool m2 = m1 && hi == mhi;
        const uint32_t lo = m2 ? (uint32_t)bk : 0u;
        const uint32_t mlo = __reduce_max_sync(0xffffffffu, lo);
        const bool m3 = m2 && lo == mlo;
        const uint32_t best = __reduce_min_sync(0xffffffffu, m3 ? bx : 0xffffffffu);
        __syncwarp();
        if (lane == 0) {
          for (uint32_t i = 0; i < sm->nsel[t]; ++i)
            if (sm->sel[t][i] == occupant) { sm->sel[t][i] = (uint8_t)best; break; }
          cnt[occupant] -= 1;
          cnt[best] += 1;
          if (sub_pos >= 0) {
            sm->sub_c[t][sub_pos] = (uint8_t)best;
          } else {
            for (uint32_t i = (uint32_t)kept_pos; i + 1 < sm->nkept[t]; ++i)
              sm->kept[t][i] = sm->kept[t][i + 1];
            sm->nkept[t] -= 1;
            const uint32_t ns = sm->nsub[t];
            sm->sub_d[t][ns] = (uint8_t)orig;
            sm->sub_c[t][ns] = (uint8_t)best;
            sm->nsub[t] = (uint8_t)(ns + 1);
          }
        }
        __syncwarp();
        selm = (selm & ~bit(occupant)) | bit(best);
        changed = true;
      }
    }
  }
}

// balancer.cpp:8-38 on warp 0. uid/batch ascending by uid on entry.
__device__ inline void balance_warp(const uint8_t* uid, const uint16_t* batch, uint32_t n,
                                    uint64_t t_cpu_token, uint64_t t_load, uint8_t* load,
                                    uint32_t& n_load, uint8_t* cpu, uint32_t& n_cpu) {
  __shared__ uint8_t sorted[kMaxE];
  const int lane = lane_id();
  for (uint32_t i = lane; i < n; i += 32) {
    uint32_t r = 0;
    for (uint32_t j = 0; j < n; ++j)
      r += batch[j] > batch[i] || (batch[j] == batch[i] && uid[j] < uid[i]);
    sorted[r] = (uint8_t)i;
  }
  __syncwarp();
  n_load = n_cpu = 0;
  uint64_t c_load = 0, c_cpu = 0;
  if (n > 0) {
    int l = 0, r = (int)n - 1;
    while (l <= r) {
      if (c_load <= c_cpu) {
        c_load += t_load;
        load[n_load++] = uid[sorted[l]];
        ++l;
      } else {
        c_cpu += (uint64_t)batch[sorted[r]] * t_cpu_token;
        cpu[n_cpu++] = uid[sorted[r]];
        if (r == 0) break;
        --r;
      }
    }
  }
  __syncwarp();
}

// --------------------------------------------------------------- step
struct StepScratch {
  uint64_t attn_end, route_end;
  uint16_t cnt[kMaxE];
  uint8_t duid[kMaxE];
  uint16_t dbat[kMaxE];
  uint32_t ndm;
};

__device__ inline void log_eviction(const Logs* lg, StepOut* out, uint64_t now, uint32_t layer,
                                    uint32_t e) {
  if (lane_id() == 0) {
    if (lg && lg->evs) {
      const unsigned long long i = atomicAdd(&lg->counts[2], 1ULL);
      if (i < lg->cap_evs) {
        EvRec r;
        r.time = now; r.layer = layer; r.e = e;
        lg->evs[i] = r;
      } else {
        *lg->overflow = 1;
      }
    }
    if (out->n_evict < 2 * kMaxE) {
      // ev_layer/ev_e live in the StepRec; StepOut keeps only the count
    }
    out->n_evict++;
  }
}

// admit_or_defer (pipeline.cpp:93-108), warp-collective. Returns the slot
// (>= 0), -1 when nothing was inserted, -2 when the admission was deferred.
__device__ inline int admit_or_defer(const StepCtx& cx, DecideSmem* sm, LayerState* ls,
                                     const double* hist, uint32_t layer, uint32_t e, uint64_t now,
                                     bool shield_it, uint8_t* ev_layer, uint8_t* ev_e,
                                     const double* avg) {
  const DevCfg& cfg = *cx.cfg;
  if (has(ls->mask, e)) return ls->slot_of[e];
  int victim, slot;
  const int rc = admit_warp(ls, hist, cfg, e, now, victim, slot, avg);
  if (rc == 3) {
    if (lane_id() == 0) sm->def_e[sm->n_def++] = e;
    __syncwarp();
    return -2;
  }
  if (rc == 4) {
    if (lane_id() == 0) cx.st->err = 4;
    return -1;
  }
  if (victim >= 0) {
    if (lane_id() == 0 && sm->out.n_evict < 2 * kMaxE) {
      ev_layer[sm->out.n_evict] = (uint8_t)layer;
      ev_e[sm->out.n_evict] = (uint8_t)victim;
    }
    __syncwarp();
    log_eviction(cx.logs, &sm->out, now, layer, (uint32_t)victim);
    __syncwarp();
  }
  if (shield_it && lane_id() == 0) ls->shield |= bit(e);
  __syncwarp();
  return slot;
}

// The step. Caller fills sm->s (and sm->ns / sm->np / sm->next_has_pred when
// cx.has_target && cfg.pre) and __syncthreads() before the call.
// The stochastic next-layer predictor (prefetch.cpp:34-83) for every token,
// the per-expert max merge (pipeline.cpp:412-425) and the build_queue
// ranking (prefetch.cpp:96-105). Independent of the executing layer's
// decisions, so the stack runs it on warp 1 while warp 0 routes.
__device__ inline void predict_queue_warp(const StepCtx& cx, DecideSmem* sm, NextSmem* nx) {
  const DevCfg& cfg = *cx.cfg;
  EngineState* st = cx.st;
  const uint32_t lane = (uint32_t)lane_id();
  const uint32_t E = cfg.E, B = cfg.B, k = cfg.k;
  // (1) lane t: argmax_first (prefetch.cpp:12-20: max value, lowest index)
  // of token t's vector — the supplied prediction, or the true next scores;
  // experts visited in a lane-rotated order (no bank conflicts), the
  // (value desc, index asc) rule makes the order irrelevant
  __shared__ uint8_t s_amax[kMaxB], s_head[kMaxB];
  if (lane < B) {
    const bool supplied = (sm->next_has_pred >> lane) & 1ULL;
    const double* v = supplied ? sm->np[lane] : sm->ns[lane];
    double bv = 0.0;
    uint32_t bi = 0xffffffffu;
    for (uint32_t j = 0; j < E; ++j) {
      uint32_t e = j + lane % E;
      if (e >= E) e -= E;
      const double x = v[e];
      if (bi == 0xffffffffu || x > bv || (x == bv && e < bi)) { bv = x; bi = e; }
    }
    s_amax[lane] = (uint8_t)bi;
  }
  __syncwarp();
  // (2) lane 0: the heads, in token order from the one predictor stream
  // (prefetch.cpp:34-83; draws only for tokens without a supplied vector)
  if (lane == 0) {
    uint64_t rs[4] = {st->rng[0], st->rng[1], st->rng[2], st->rng[3]};
    Counters& c = st->c;
    for (uint32_t t = 0; t < B; ++t) {
      const uint64_t ntop = nx->top[t], nact = nx->act[t];
      uint32_t head;
      int kind;
      if ((sm->next_has_pred >> t) & 1ULL) {
        head = s_amax[t];
        kind = has(ntop, head) ? 0 : (has(nact, head) ? 1 : 2);
        c.trace_supplied++;
      } else {
        const uint32_t n_top = __popcll(ntop);
        if (rng_double(rs) < cfg.p_top && n_top > 0) {
          uint32_t pick = rng_below_small(rs, n_top);
          head = 0;
          for (uint32_t r = 0; r < k; ++r) {
            const uint32_t e = nx->order[t][r];
            if (has(ntop, e) && pick-- == 0) { head = e; break; }
          }
          kind = 0;
        } else {
          const uint64_t lows = nact & ~ntop;
          const uint32_t n_low = __popcll(lows);
          if (rng_double(rs) < cfg.p_active && n_low > 0) {
            uint32_t pick = rng_below_small(rs, n_low);
            head = 0;
            for (uint32_t r = 0; r < k; ++r) {
              const uint32_t e = nx->order[t][r];
              if (has(lows, e) && pick-- == 0) { head = e; break; }
            }
            kind = 1;
          } else {
            const uint64_t allm = E >= 64 ? ~0ULL : ((1ULL << E) - 1ULL);
            const uint64_t inact = allm & ~nact;
            uint32_t pick = rng_below_small(rs, __popcll(inact));
            uint64_t m = inact;
            for (uint32_t i = 0; i < pick; ++i) m &= m - 1;
            head = __ffsll((long long)m) - 1;
            kind = 2;
          }
        }
        c.draws++;
      }
      if (kind == 0) c.head_top++; else if (kind == 1) c.head_active++; else c.head_inactive++;
      s_head[t] = (uint8_t)head;
    }
    st->rng[0] = rs[0]; st->rng[1] = rs[1]; st->rng[2] = rs[2]; st->rng[3] = rs[3];
  }
  __syncwarp();
  // (3) lane-per-expert merge: elementwise max over tokens (pipeline.cpp:
  // 412-425) of each token's predicted vector — supplied verbatim, or the
  // true vector with the head and the true argmax swapped
  for (uint32_t e = lane; e < E; e += 32) {
    double m = 0.0;
    for (uint32_t t = 0; t < B; ++t) {
      double v;
      if ((sm->next_has_pred >> t) & 1ULL) {
        v = sm->np[t][e];
      } else {
        const double* tn = sm->ns[t];
        const uint32_t head = s_head[t], tt = s_amax[t];
        v = (e == head) ? tn[tt] : ((e == tt) ? tn[head] : tn[e]);
      }
      if (m < v) m = v;
    }
    sm->merged[e] = m;
  }
  __syncwarp();
  // build_queue (prefetch.cpp:85-115): rank merged, first `depth` non-resident
  uint8_t* qorder = sm->qorder;
  for (uint32_t e = lane; e < E; e += 32) {
    const double v = sm->merged[e];
    uint32_t r = 0;
    for (uint32_t j = 0; j < E; ++j) {
      const double vj = sm->merged[j];
      r += (vj > v) || (vj == v && j < e);
    }
    qorder[r] = (uint8_t)e;
  }
  __syncwarp();
}

// The previous step's schedule_prefetch (pipeline.cpp:293-344) into THIS
// layer, run by warp 0 at the start of this step in predictor mode: the
// same state transition as at the end of the previous step (nothing happens
// in between in the reference's state machine), with every token's
// prediction supplied (prefetch.cpp:43-49: verbatim, head = first argmax,
// RNG untouched) and the head kinds counted against this step's true scores.
// Issues, evictions and the queue go to the previous step's record.
__device__ inline void deferred_prefetch(const StepCtx& cx, DecideSmem* sm, uint8_t* ev_layer, uint8_t* ev_e) {
  const DevCfg& cfg = *cx.cfg;
  EngineState* st = cx.st;
  const uint32_t lane = (uint32_t)lane_id();
  const uint32_t E = cfg.E, B = cfg.B, layer = cx.layer;
  const uint64_t it = cx.it;
  LayerState* ls = cx.ls;
  // heads (lane t) and their kinds, then the per-expert max merge
  __shared__ uint8_t s_kind[kMaxB];
  if (lane < B) {
    const double* v = sm->np[lane];
    double bv = 0.0;
    uint32_t bi = 0xffffffffu;
    for (uint32_t j = 0; j < E; ++j) {
      uint32_t e = j + lane % E;
      if (e >= E) e -= E;
      const double x = v[e];
      if (bi == 0xffffffffu || x > bv || (x == bv && e < bi)) { bv = x; bi = e; }
    }
    s_kind[lane] = has(sm->top[lane], bi) ? 0 : (has(sm->act[lane], bi) ? 1 : 2);
  }
  for (uint32_t e = lane; e < E; e += 32) {
    double m = 0.0;
    for (uint32_t t = 0; t < B; ++t) m = m < sm->np[t][e] ? sm->np[t][e] : m;
    sm->merged[e] = m;
  }
  __syncwarp();
  if (lane == 0) {
    Counters& c = st->c;
    for (uint32_t t = 0; t < B; ++t) {
      c.trace_supplied++;
      if (s_kind[t] == 0) c.head_top++; else if (s_kind[t] == 1) c.head_active++; else c.head_inactive++;
    }
  }
  uint8_t* qorder = sm->qorder;
  for (uint32_t e = lane; e < E; e += 32) {
    const double v = sm->merged[e];
    uint32_t r = 0;
    for (uint32_t j = 0; j < E; ++j) {
      const double vj = sm->merged[j];
      r += (vj > v) || (vj == v && j < e);
    }
    qorder[r] = (uint8_t)e;
  }
  __syncwarp();
  // build_queue + issue against the gate of this layer (completion of the
  // previous step + t_attn), from max(pcie_free, its resident_done)
  const uint64_t gate = st->now + cfg.t_attn;
  uint32_t qn = 0;
  uint8_t qe[kMaxE];
  if (cfg.depth > 0)
    for (uint32_t r = 0; r < E && qn < cfg.depth; ++r) {
      const uint32_t e = qorder[r];
      if (!has(ls->mask, e)) qe[qn++] = (uint8_t)e;
    }
  uint64_t t = st->pcie_free > st->pf_resident_done ? st->pcie_free : st->pf_resident_done;
  uint64_t issued = 0;
  uint32_t n_pref = 0;
  bool avg_done = false;
  for (uint32_t i = 0; i < qn; ++i) {
    if (t + cfg.t_load > gate) break;
    const uint32_t e = qe[i];
    if (has(ls->mask, e)) continue;
    t += cfg.t_load;
    issued |= bit(i);
    if (!avg_done && cfg.policy == 0) {  // this layer's averages before this step records
      for (uint32_t x = lane; x < E; x += 32) sm->tavg[x] = window_average(ls, cx.hist_l, cfg.window, E, x);
      __syncwarp();
      avg_done = true;
    }
    const int slot = admit_or_defer(cx, sm, ls, cx.hist_l, layer, e, t, false, ev_layer, ev_e, sm->tavg);
    if (lane == 0) {
      sm->out.pref[n_pref] = (uint8_t)e;
      sm->out.pref_slot[n_pref] = (int8_t)(slot >= 0 ? slot : -1);
    }
    ++n_pref;
    __syncwarp();
  }
  __syncwarp();  // every lane has read pcie_free
  if (lane == 0) {
    if (t > st->pcie_free) st->pcie_free = t;
    st->q_valid = 1;
    st->q_layer = layer;
    st->q_it = it;
    st->q_n = qn;
    st->q_issued = issued;
    for (uint32_t i = 0; i < qn; ++i) st->q_e[i] = qe[i];
    st->c.issued += n_pref;
    st->c.prefetch += n_pref;
    sm->out.pref_layer = layer;
    sm->out.n_pref = n_pref;
    st->pf_pending = 0;
  }
  __syncwarp();
}

// Called by warp 0 as soon as the demand-load / BA-stream lists are final
// (before the GPU task clock, deferrals and prefetch), so the caller can hand
// the uploads to the copy engine early.
// classified(): called by warp 2 right after classification, concurrently with
// routing on warp 0, with the pre-route residency snapshot — the stack
// publishes the experts certain to be selected there (speculative FFN start).
// plan_ready(): called by warp 0 once the executing layer's outcome (hits,
// loads, BA split, deferred admissions) is final, before the prefetch phase.
struct NoHook {
  __device__ void operator()(DecideSmem*, uint32_t, uint32_t) const {}
  __device__ void classified(DecideSmem*, uint64_t) const {}
  __device__ void classified_early(DecideSmem*, uint64_t) const {}
  __device__ void plan_ready(DecideSmem*) const {}
  __device__ void prefetched(DecideSmem*) const {}
};

template <class Hook = NoHook>
__device__ inline void decide_step(const StepCtx& cx, DecideSmem* sm, NextSmem* nx,
                                   StepScratch* sc, StepRec* rec_out, TokRec* tok_out,
                                   const Hook& on_loads = Hook()) {
  const DevCfg& cfg = *cx.cfg;
  EngineState* st = cx.st;
  const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const uint32_t E = cfg.E, B = cfg.B, k = cfg.k, layer = cx.layer;
  const uint64_t it = cx.it;

  const uint32_t nw = blockDim.x >> 5;
#ifdef MOEB_PROFILE_PHASES
  uint64_t tp = (cx.prof && tid == 0) ? ptimer() : 0;
  auto mark = [&](int i) {
    if (cx.prof && tid == 0) { const uint64_t n = ptimer(); cx.prof[i] += n - tp; tp = n; }
  };
#else
  auto mark = [](int) {};  // phase timers compiled out (build with -DMOEB_PROFILE_PHASES)
#endif
  if (tid == 0) {
    sm->n_def = 0;
    sm->out.n_load = sm->out.n_cpu = sm->out.n_pref = sm->out.n_def = sm->out.n_evict = 0;
    sm->out.n_res = 0;
  }
  // classify every token (and the prefetch target's tokens) — warp per token
  const bool want_next = cfg.pre && cx.has_target && !cx.defer_prefetch;
  // this step's tokens now; the prefetch target's tokens (only the predictor
  // on warp 1 needs them) are classified after the fork by warps 4..
  for (uint32_t t = warp; t < B; t += nw) {
    uint64_t a, tp, lw, al;
    double b, T, L, R;
    classify_warp(sm->s[t], E, k, cfg.alpha, sm->order[t], a, tp, lw, al, b, T, L, R, cx.f32_scores != 0);
    if (lane == 0) {
      sm->act[t] = a; sm->top[t] = tp; sm->low[t] = lw; sm->alt[t] = al;
      sm->beta[t] = b; sm->thT[t] = T; sm->thL[t] = L; sm->thR[t] = R;
    }
  }
  __syncthreads();
  // predictor mode: the previous step's prefetch into this layer first (its
  // admissions are part of the residency this step's router sees)
  __shared__ uint8_t pev_layer[2 * kMaxE], pev_e[2 * kMaxE];
  if (cx.run_pending && warp == 0) {
    StepRec* pr = cx.prev_rec;
    uint32_t n0 = pr ? pr->n_evict : 0u;
    if (lane == 0) sm->out.n_evict = n0;  // append to the previous step's evictions
    __syncwarp();
    deferred_prefetch(cx, sm, pev_layer, pev_e);
    const uint32_t n1 = sm->out.n_evict < 2 * kMaxE ? sm->out.n_evict : 2 * kMaxE;
    if (pr) {
      for (uint32_t i = n0 + lane; i < n1; i += 32) {
        pr->ev_layer[i] = pev_layer[i];
        pr->ev_e[i] = pev_e[i];
      }
      for (uint32_t i = lane; i < sm->out.n_pref; i += 32) pr->pref[i] = sm->out.pref[i];
      if (lane == 0) {
        pr->n_evict = (uint8_t)n1;
        pr->n_pref = (uint8_t)sm->out.n_pref;
      }
    }
    __syncwarp();
    if (lane == 0) sm->out.n_evict = 0;
  }
  // predictor mode: the previous step's prefetch commands go out now (warp 0)
  if (cx.defer_prefetch && warp == 0) on_loads.prefetched(sm);
  if (tid == 0) {
    const uint64_t start = st->now;
    // attention + gate (pipeline.cpp:133-145)
    const uint64_t attn_end = start + cfg.t_attn;
    log_task(cx.logs, R_GPU, K_ATTN, -1, 0, start, attn_end, layer, it);
    st->gpu_free = attn_end;
    if (st->q_valid && st->q_layer == layer && st->q_it == it) {
      const uint64_t all = st->q_n >= 64 ? ~0ULL : ((1ULL << st->q_n) - 1ULL);
      st->c.cancelled += __popcll(all & ~st->q_issued);
      st->q_valid = 0;
    }
    // routing on CPU (pipeline.cpp:147-152)
    const uint64_t route_start = attn_end > st->cpu_free ? attn_end : st->cpu_free;
    const uint64_t route_end = route_start + cfg.t_route;
    log_task(cx.logs, R_CPU, K_ROUTE, -1, 0, route_start, route_end, layer, it);
    st->cpu_free = route_end;
    sc->attn_end = attn_end;
    sc->route_end = route_end;
  }
  __syncthreads();
  const uint64_t mask = cx.ls->mask;  // snapshot the router sees (pipeline.cpp:154-155)
  __syncthreads();
  mark(4);
  // the speculative plan needs only the classification and the snapshot:
  // built by the last warp beside route pass 2 when that warp routes no
  // token; the route barrier below then leaves that warp out (it hands its
  // result to warp 2 on named barrier 7), so route -> loads -> mailbox A on
  // warp 0 never waits for it
  const bool early_spec = B < nw && nw >= 5;
  if (early_spec && warp == (int)nw - 1) {
    on_loads.classified_early(sm, mask);
    asm volatile("bar.arrive 7, 64;" ::: "memory");
  }
  // route pass 2 (router.cpp:114-149), one warp per token; C (the union of
  // the batch's top-score experts, router.cpp:105-112) computed by every warp
  if (cfg.er) {
    uint64_t C = 0;
    for (uint32_t t = 0; t < B; ++t) C |= sm->top[t];
    if (tid == 0) sm->C = C;
    for (uint32_t t = warp; t < B; t += nw) route_token_warp(sm, t, mask, E, k, C);
  } else {
    // plain_top_k (router.cpp:35-39)
    for (uint32_t t = warp; t < B; t += nw) {
      if ((uint32_t)lane < k) sm->sel[t][lane] = sm->order[t][lane];
      if (lane == 0) {
        sm->nsel[t] = (uint8_t)k;
        sm->nsub[t] = 0;
        sm->nkept[t] = 0;
      }
    }
  }
  if (early_spec) {
    if (warp != (int)nw - 1) asm volatile("bar.sync 6, %0;" ::"r"((nw - 1) * 32) : "memory");
  } else {
    __syncthreads();
  }
  mark(17);

  // ---- fork. warp 0 routes and runs the order-dependent rest; alongside it
  //   warp 1: the next-layer predictor + queue ranking (barrier 2),
  //   warp 2: the speculative plan of the certain experts (hook; barrier 3),
  //   warp 3: mean scores -> record_scores -> window averages (barrier 4).
  // record_scores (pipeline.cpp:191) reads only this step's scores and
  // nothing before the first admission reads the history, so recording it
  // beside the routing is the same computation as recording it after.
  const bool want_pred = want_next;
  const uint32_t nx_threads = (nw - 4 + 1) * 32;  // warps 4.. + warp 1 (barrier 5)
  if (warp >= 4) {
    if (want_pred) {
      for (uint32_t t = warp - 4; t < B; t += nw - 4) {
        uint64_t a, tp, lw, al;
        double b, T, L, R;
        classify_warp(sm->ns[t], E, k, cfg.alpha, nx->order[t], a, tp, lw, al, b, T, L, R, cx.f32_scores != 0);
        if (lane == 0) { nx->act[t] = a; nx->top[t] = tp; }
      }
      asm volatile("bar.arrive 5, %0;" ::"r"(nx_threads) : "memory");
    }
    return;
  }
  if (warp == 1) {
    if (want_pred) {
      asm volatile("bar.sync 5, %0;" ::"r"(nx_threads) : "memory");  // the target's classification
      predict_queue_warp(cx, sm, nx);
      asm volatile("bar.arrive 2, 64;" ::: "memory");
    }
    return;
  }
  if (warp == 2) {
    if (early_spec) asm volatile("bar.sync 7, 64;" ::: "memory");  // the last warp's speculative plan
    on_loads.classified(sm, mask);
    asm volatile("bar.arrive 3, 64;" ::: "memory");
    return;
  }
  if (warp == 3) {
    // mean over tokens in token order (pipeline.cpp:79-91)
    for (uint32_t e = lane; e < E; e += 32) {
      double m = 0.0;
      for (uint32_t t = 0; t < B; ++t) m += sm->s[t][e];
      sm->mean[e] = m / (double)B;
    }
    __syncwarp();
    record_scores_warp(cx.ls, cx.hist_l, cfg.window, E, sm->mean);
    if (cfg.policy == 0) {
      // window averages of the executing layer (after recording) and of the
      // prefetch target (unchanged by this step unless it is this layer)
      for (uint32_t e = lane; e < E; e += 32) {
        sm->avg[e] = window_average(cx.ls, cx.hist_l, cfg.window, E, e);
        if (want_next && cx.tls != cx.ls) sm->tavg[e] = window_average(cx.tls, cx.thist, cfg.window, E, e);
      }
    }
    asm volatile("bar.arrive 4, 64;" ::: "memory");
    return;
  }
  if (warp != 0) return;  // the rest is order-dependent: warp 0 in lock-step

  // coalescing is a no-op for a single token: every candidate's batch count
  // is 0, never above the occupant's (router.cpp:203-228)
  if (cfg.er && B > 1) coalesce_warp(sm, B, E, k, mask, sc->cnt);
  __syncwarp();
  mark(5);

  // ---- hit accounting + batch_of (pipeline.cpp:176-189)
  // lane t <-> token t (B <= 32): selection masks, counts by ballot
  uint64_t n_sel_total = 0, n_hits = 0, n_subs = 0, n_kept = 0;
  {
    uint64_t m = 0;
    uint32_t ns = 0, nb = 0, nk = 0;
    if ((uint32_t)lane < B) {
      ns = sm->nsel[lane];
      for (uint32_t i = 0; i < ns; ++i) m |= bit(sm->sel[lane][i]);
      nb = sm->nsub[lane];
      nk = sm->nkept[lane];
    }
    n_sel_total = __reduce_add_sync(0xffffffffu, ns);
    n_hits = __reduce_add_sync(0xffffffffu, (uint32_t)__popcll(m & mask));
    n_subs = __reduce_add_sync(0xffffffffu, nb);
    n_kept = __reduce_add_sync(0xffffffffu, nk);
    batch_counts(m, B, E, sc->cnt);
  }
  mark(28);
  if (lane == 0) {
    Counters& c = st->c;
    if (cfg.er) { c.subs += n_subs; c.kept_low += n_kept; }
    c.selections += n_sel_total;
    c.hits += n_hits;
    c.misses += n_sel_total - n_hits;
  }
  LayerState* ls = cx.ls;
  double* hist_l = cx.hist_l;
  // window averages: warp 3 recorded this step's mean and computed them
  bool avg_ready = false;
  auto avg = [&]() -> const double* {
    if (!avg_ready) {
      asm volatile("bar.sync 4, 64;" ::: "memory");
      avg_ready = true;
    }
    return sm->avg;
  };
  mark(29);

  // residents: shield + touch; misses -> demand set (pipeline.cpp:196-205)
  const uint64_t route_end = sc->route_end, attn_end = sc->attn_end;
  const bool c0 = (uint32_t)lane < E && sc->cnt[lane] > 0;
  const bool c1 = (uint32_t)lane + 32 < E && sc->cnt[lane + 32] > 0;
  const uint64_t distinct = ballot64(c0, c1);
  const uint64_t res_sel = distinct & mask;
  const uint64_t miss = distinct & ~mask;
  {
    // lists in ascending expert order: lane l places experts l and l + 32 by
    // a popcount of the lower set bits
    auto place = [&](uint32_t e) {
      if (has(res_sel, e)) {
        ls->last_access[e] = route_end;
        const uint32_t i = (uint32_t)__popcll(res_sel & (bit(e) - 1ULL));
        sm->out.res_slot[i] = ls->slot_of[e];
        sm->out.res[i] = (uint8_t)e;
      } else if (has(miss, e)) {
        const uint32_t i = (uint32_t)__popcll(miss & (bit(e) - 1ULL));
        sc->duid[i] = (uint8_t)e;
        sc->dbat[i] = sc->cnt[e];
      }
    };
    if ((uint32_t)lane < E) place(lane);
    if ((uint32_t)lane + 32 < E) place(lane + 32);
  }
  if (lane == 0) {
    ls->shield |= res_sel;
    sc->ndm = (uint32_t)__popcll(miss);
    sm->out.n_res = (uint32_t)__popcll(res_sel);
    sm->out.res_mask = res_sel;
    sm->out.mask_before = mask;
  }
  for (uint32_t e = lane; e < E; e += 32) sm->out.cnt[e] = sc->cnt[e];
  __syncwarp();

  mark(6);
  // BA split (pipeline.cpp:207-215)
  uint32_t n_load = 0, n_cpu = 0;
  if (cfg.ba) {
    balance_warp(sc->duid, sc->dbat, sc->ndm, cfg.t_cpu_token, cfg.t_load, sm->out.load, n_load,
                 sm->out.cpu, n_cpu);
  } else {
    if (lane == 0)
      for (uint32_t i = 0; i < sc->ndm; ++i) sm->out.load[i] = sc->duid[i];
    n_load = sc->ndm;
    n_cpu = 0;
  }
  __syncwarp();
  mark(18);

  // the per-step record's eviction arrays double as scratch for StepOut
  __shared__ uint8_t ev_layer[2 * kMaxE], ev_e[2 * kMaxE];

  // CPU expert tasks (pipeline.cpp:217-227)
  uint64_t cpu_t = route_end > st->cpu_free ? route_end : st->cpu_free;
  for (uint32_t i = 0; i < n_cpu; ++i) {
    const uint32_t e = sm->out.cpu[i];
    const uint64_t dur = (uint64_t)sc->cnt[e] * cfg.t_cpu_token;
    if (lane == 0) log_task(cx.logs, R_CPU, K_CPU, (int)layer, e, cpu_t, cpu_t + dur, layer, it);
    cpu_t += dur;
  }
  __syncwarp();  // every lane has read cpu_free
  if (lane == 0) { st->cpu_free = cpu_t; st->c.cpu_computed += n_cpu; }
  __syncwarp();
  mark(19);

  // demand loads, serial on PCIe, admitted + shielded (pipeline.cpp:229-240)
  uint64_t ready[kMaxE];
  uint64_t pcie_t = route_end > st->pcie_free ? route_end : st->pcie_free;
  for (uint32_t i = 0; i < n_load; ++i) {
    const uint32_t e = sm->out.load[i];
    if (lane == 0) log_task(cx.logs, R_PCIE, K_DEMAND, (int)layer, e, pcie_t, pcie_t + cfg.t_load, layer, it);
    pcie_t += cfg.t_load;
    const int slot = admit_or_defer(cx, sm, ls, hist_l, layer, e, pcie_t, true, ev_layer, ev_e, avg());
    if (lane == 0) sm->out.load_slot[i] = (int8_t)(slot >= 0 ? slot : -1);
    ready[i] = pcie_t;
  }
  __syncwarp();  // every lane has read pcie_free
  if (lane == 0) { st->pcie_free = pcie_t; st->c.demand += n_load; }
  __syncwarp();
  mark(20);
  on_loads(sm, n_load, n_cpu);
  mark(21);

  // GPU expert compute (pipeline.cpp:242-266)
  uint64_t gpu_t = st->gpu_free > route_end ? st->gpu_free : route_end;
  uint64_t resident_done = attn_end > route_end ? attn_end : route_end;
  const uint32_t nres = sm->out.n_res;
  for (uint32_t i = 0; i < nres; ++i) {
    if (lane == 0) log_task(cx.logs, R_GPU, K_RESIDENT, (int)layer, sm->out.res[i], gpu_t, gpu_t + cfg.t_gpu, layer, it);
    gpu_t += cfg.t_gpu;
  }
  if (nres) resident_done = gpu_t;
  for (uint32_t i = 0; i < n_load; ++i) {
    const uint64_t s0 = gpu_t > ready[i] ? gpu_t : ready[i];
    if (lane == 0) log_task(cx.logs, R_GPU, K_LOADED, (int)layer, sm->out.load[i], s0, s0 + cfg.t_gpu, layer, it);
    gpu_t = s0 + cfg.t_gpu;
  }
  uint64_t completion = attn_end;
  if (route_end > completion) completion = route_end;
  if (cpu_t > completion) completion = cpu_t;
  if ((nres || n_load) && gpu_t > completion) completion = gpu_t;
  __syncwarp();  // every lane has read gpu_free
  if (lane == 0) {
    st->gpu_free = gpu_t;
    const Logs* lg = cx.logs;
    if (lg && lg->wins) {
      const unsigned long long i = atomicAdd(&lg->counts[1], 1ULL);
      if (i < lg->cap_wins) {
        WinRec w;
        w.it = it; w.layer = layer; w.pad = 0; w.attn_end = attn_end; w.route_end = route_end;
        w.completion = completion; w.sel = distinct;
        lg->wins[i] = w;
      } else {
        *lg->overflow = 1;
      }
    }
    sm->out.n_load = n_load;
    sm->out.n_cpu = n_cpu;
    ls->shield = 0;  // unshield_layer (pipeline.cpp:276)
  }
  __syncwarp();
  mark(22);

  // warp 2's speculative plan is out (it read the slots of shielded hits,
  // which a deferred admission below may now evict)
  asm volatile("bar.sync 3, 64;" ::: "memory");
  // deferred admissions, FIFO, unshielded, at completion (pipeline.cpp:277-280)
  {
    const uint32_t nd = sm->n_def;
    uint32_t def_copy[2 * kMaxE];
    for (uint32_t i = 0; i < nd; ++i) def_copy[i] = sm->def_e[i];
    __syncwarp();
    if (lane == 0) sm->n_def = 0;
    __syncwarp();
    for (uint32_t i = 0; i < nd; ++i) {
      const int slot = admit_or_defer(cx, sm, ls, hist_l, layer, def_copy[i], completion, false, ev_layer, ev_e, avg());
      if (lane == 0 && slot >= 0 && sm->out.n_def < kMaxE) {
        sm->out.def_e[sm->out.n_def] = (uint8_t)def_copy[i];
        sm->out.def_slot[sm->out.n_def] = (int8_t)slot;
        sm->out.n_def++;
      }
      __syncwarp();
    }
  }
  if (lane == 0) sm->out.completion = completion;
  __syncwarp();
  mark(23);
  on_loads.plan_ready(sm);

  mark(7);
  // prefetch for the next layer (pipeline.cpp:293-344)
  uint32_t n_pref = 0;
  if (want_next) {
    const uint32_t tl = cx.target_layer;
    const uint64_t tit = cx.target_it;
    const uint64_t gate = completion + cfg.t_attn;
    LayerState* tls = cx.tls;
    const double* tavg = nullptr;  // warp 3's averages of the target layer
    asm volatile("bar.sync 2, 64;" ::: "memory");  // warp 1's predictor + queue ranking
    const uint8_t* qorder = sm->qorder;
    const uint64_t tmask = tls->mask;
    uint32_t qn = 0;
    uint8_t qe[kMaxE];
    if (cfg.depth > 0)
      for (uint32_t r = 0; r < E && qn < cfg.depth; ++r) {
        const uint32_t e = qorder[r];
        if (!has(tmask, e)) qe[qn++] = (uint8_t)e;
      }
    uint64_t t = st->pcie_free > resident_done ? st->pcie_free : resident_done;
    uint64_t issued = 0;
    for (uint32_t i = 0; i < qn; ++i) {
      if (t + cfg.t_load > gate) break;
      const uint32_t e = qe[i];
      if (has(tls->mask, e)) continue;
      if (lane == 0) log_task(cx.logs, R_PCIE, K_PREFETCH, (int)tl, e, t, t + cfg.t_load, tl, tit);
      t += cfg.t_load;
      issued |= bit(i);
      if (!tavg && cfg.policy == 0) tavg = (tl == layer) ? avg() : (avg(), sm->tavg);
      const int slot = admit_or_defer(cx, sm, tls, cx.thist, tl, e, t, false, ev_layer, ev_e, tavg);
      if (lane == 0) {
        sm->out.pref[n_pref] = (uint8_t)e;
        sm->out.pref_slot[n_pref] = (int8_t)(slot >= 0 ? slot : -1);
      }
      ++n_pref;
      __syncwarp();
    }
    __syncwarp();  // every lane has read pcie_free
    if (lane == 0) {
      if (t > st->pcie_free) st->pcie_free = t;
      st->q_valid = 1;
      st->q_layer = tl;
      st->q_it = tit;
      st->q_n = qn;
      st->q_issued = issued;
      for (uint32_t i = 0; i < qn; ++i) st->q_e[i] = qe[i];
      st->c.issued += n_pref;
      st->c.prefetch += n_pref;
      sm->out.pref_layer = tl;
    }
    __syncwarp();
  }
  mark(8);
  avg();  // warp 3 has recorded this step's scores (and retired)
  if (lane == 0 && cx.defer_prefetch) {
    // predictor mode: this step's schedule_prefetch runs at the start of the
    // next step (which has the prediction); nothing past the trace end
    st->pf_pending = (cfg.pre && cx.has_target) ? 1u : 0u;
    st->pf_layer = cx.target_layer;
    st->pf_it = cx.target_it;
    st->pf_resident_done = resident_done;
  }
  if (lane == 0) {
    sm->out.n_pref = n_pref;
    sm->out.completion = completion;
    sm->out.resident_done = resident_done;
    st->now = completion;
  }
  __syncwarp();

  // per-step decision record
  if (rec_out) {
    if (lane == 0) {
      rec_out->it = it;
      rec_out->layer = layer;
      rec_out->B = B;
      rec_out->mask_before = mask;
      rec_out->completion = completion;
      rec_out->n_load = (uint8_t)n_load;
      rec_out->n_cpu = (uint8_t)n_cpu;
      rec_out->n_pref = (uint8_t)n_pref;
      rec_out->n_evict = (uint8_t)(sm->out.n_evict < 2 * kMaxE ? sm->out.n_evict : 2 * kMaxE);
    }
    for (uint32_t i = lane; i < n_load; i += 32) rec_out->load[i] = sm->out.load[i];
    for (uint32_t i = lane; i < n_cpu; i += 32) rec_out->cpu[i] = sm->out.cpu[i];
    for (uint32_t i = lane; i < n_pref; i += 32) rec_out->pref[i] = sm->out.pref[i];
    for (uint32_t i = lane; i < sm->out.n_evict && i < 2 * kMaxE; i += 32) {
      rec_out->ev_layer[i] = ev_layer[i];
      rec_out->ev_e[i] = ev_e[i];
    }
    for (uint32_t t = lane; t < B; t += 32) {
      TokRec& tr = tok_out[t];
      tr.n_sel = sm->nsel[t];
      tr.n_sub = sm->nsub[t];
      tr.n_kept = sm->nkept[t];
      for (uint32_t i = 0; i < sm->nsel[t]; ++i) tr.sel[i] = sm->sel[t][i];
      for (uint32_t i = 0; i < sm->nsub[t]; ++i) { tr.sub_d[i] = sm->sub_d[t][i]; tr.sub_c[i] = sm->sub_c[t][i]; }
      for (uint32_t i = 0; i < sm->nkept[t]; ++i) tr.kept[i] = sm->kept[t][i];
    }
  }
  __syncwarp();
}

}  // namespace moeb
