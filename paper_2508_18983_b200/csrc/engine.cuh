// engine.cuh — device-resident decision state machine (sm_100a).
//
// One CTA of kWarps warps executes one (iteration, layer) decision step of
// the reference's Simulator::run_layer (/root/reference/proj/src/
// pipeline.cpp:128-286) plus schedule_prefetch (:293-344), bit-exactly:
//   * token-parallel phases (classify, route pass 2, predictor classify) run
//     one warp per token, lanes over experts (E <= 64: expert e lives in lane
//     e & 31, slot e >> 5);
//   * order-dependent phases (coalesce fixed point, cache admission/eviction,
//     balance, virtual clocks, prefetch issue) run on warp 0 in lock-step,
//     with warp-collective argmin/argmax helpers whose tie rules reproduce the
//     reference's ascending scans.
// Residency, shields, activity bands and selections are 64-bit masks.
#pragma once

#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

namespace moeb {

constexpr int kMaxE = 64;
constexpr int kMaxK = 16;
constexpr int kMaxB = 32;
constexpr int kMaxSlots = 64;
constexpr int kWarps = 32;
constexpr int kThreads = kWarps * 32;

// Task kinds / resources, numbering of pipeline.hpp:16-25.
enum : uint8_t { R_GPU = 0, R_CPU = 1, R_PCIE = 2 };
enum : uint8_t { K_ATTN = 0, K_ROUTE, K_RESIDENT, K_LOADED, K_CPU, K_DEMAND, K_PREFETCH };

// Decision-relevant configuration (SimConfig, core.hpp:94-106).
struct DevCfg {
  uint32_t L, E, k, B;
  double alpha;
  uint32_t slots, window;
  int32_t policy;  // effective policy: CE off => LRU (pipeline.cpp:64-70)
  int32_t er, pre, ba;
  uint64_t t_attn, t_gpu, t_cpu_token, t_load, t_route;
  double p_top, p_active;
  uint32_t depth;  // effective queue depth (core.hpp:103-105)
  uint32_t pad;
};

// CacheState::Layer (cache.hpp:67-73) + physical slot table.
struct LayerState {
  uint64_t mask;    // resident set
  uint64_t shield;  // shielded set
  uint32_t n_res, h_head, h_size, pad0;
  uint64_t last_access[kMaxE];
  int8_t slot_of[kMaxE];           // physical cache slot of a resident expert
  int8_t expert_of_slot[kMaxSlots];
  uint32_t slot_copy[kMaxSlots];   // id of the upload that last filled the slot
};

struct Counters {
  uint64_t demand, prefetch, cpu_computed, hits, misses, subs, kept_low, selections;
  uint64_t draws, trace_supplied, head_top, head_active, head_inactive, issued, cancelled;
};

struct EngineState {
  uint64_t gpu_free, cpu_free, pcie_free, now;
  uint64_t rng[4];                 // predictor stream (pipeline.cpp:62)
  uint32_t q_valid, q_layer;       // PrefetchQueue (prefetch.hpp:39-52)
  uint64_t q_it;
  uint32_t q_n, pad1;
  uint64_t q_issued;
  uint8_t q_e[kMaxE];
  Counters c;
  uint32_t next_copy;              // upload id allocator (stack mode)
  uint32_t err;                    // sticky device error (1 config, 4 logic)
  uint64_t it;                     // decode iteration (stack mode)
  uint64_t seq;                    // layer-step sequence number (stack mode)
  uint64_t ffn_bytes;              // algorithmic FFN bytes planned (stack mode)
  uint64_t ffn_launches;
  uint64_t prof[32];               // phase timers of the decision launch (ns, summed)
  uint64_t ack_cache;              // last mailbox acknowledgement seen (stack mode)
  uint32_t pf_pending, pf_layer;   // predictor mode: a schedule_prefetch awaits its prediction
  uint64_t pf_it, pf_resident_done;
  // speculative uploads (stack mode, physical only — decisions unchanged):
  // buffer b holds (or is receiving) expert sp_expert[b] of (sp_it[b], sp_layer[b])
  uint32_t sp_gen_next, sp_valid[2], sp_layer[2], sp_expert[2], sp_gen[2], sp_pad;
  uint64_t sp_it[2];
  uint64_t sp_jobs, sp_hits;
};

// Log records (layouts == moeb_task / moeb_window / moeb_eviction).
struct TaskRec {
  uint8_t res, kind;
  int16_t el;
  uint32_t e;
  uint64_t start, end;
  uint32_t layer, pad;
  uint64_t it;
};
struct WinRec {
  uint64_t it;
  uint32_t layer, pad;
  uint64_t attn_end, route_end, completion;
  uint64_t sel;
};
struct EvRec {
  uint64_t time;
  uint32_t layer, e;
};
// Per-step decision record (tokens follow in TokRec[B]).
struct StepRec {
  uint64_t it;
  uint32_t layer, B;
  uint64_t mask_before, completion;
  uint8_t n_load, n_cpu, n_pref, n_evict;
  uint8_t load[kMaxE], cpu[kMaxE], pref[kMaxE];
  uint8_t ev_layer[2 * kMaxE], ev_e[2 * kMaxE];
};
struct TokRec {
  uint8_t n_sel, n_sub, n_kept, pad;
  uint8_t sel[kMaxK], sub_d[kMaxK], sub_c[kMaxK], kept[kMaxK];
};

struct Logs {
  TaskRec* tasks;
  WinRec* wins;
  EvRec* evs;
  StepRec* steps;
  TokRec* toks;
  unsigned long long* counts;  // [0] tasks [1] wins [2] evs [3] steps
  uint64_t cap_tasks, cap_wins, cap_evs, cap_steps;
  uint32_t* overflow;
};

// Per-step physical outcome (consumed by the stack's plan builder).
struct StepOut {
  uint32_t n_load, n_cpu, n_pref, n_def, n_evict, n_res;
  uint8_t load[kMaxE];
  int8_t load_slot[kMaxE];   // -1: not admitted now (deferred / zero-slot) -> staging
  uint8_t cpu[kMaxE];
  uint8_t pref[kMaxE];
  int8_t pref_slot[kMaxE];
  uint8_t def_e[kMaxE];
  int8_t def_slot[kMaxE];    // admitted at completion; staging -> slot copy
  uint8_t res[kMaxE];        // resident (hit) experts, ascending
  int8_t res_slot[kMaxE];    // their slots at route time (a completion-time
                             // deferred admission may evict a hit afterwards)
  uint32_t pref_layer;
  uint64_t mask_before, completion, resident_done;
  uint64_t res_mask;         // the hits (set of out.res)
  uint16_t cnt[kMaxE];       // tokens per distinct selected expert
};

// Shared-memory workspace of the decision CTA.
struct DecideSmem {
  double s[kMaxB][kMaxE];    // this step's scores
  double ns[kMaxB][kMaxE];   // prefetch target's true scores
  double np[kMaxB][kMaxE];   // supplied predictions (optional)
  double merged[kMaxE];
  double mean[kMaxE];
  uint8_t qorder[kMaxE];     // merged-prediction ranking of the prefetch target
  double avg[kMaxE];         // window averages of the executing layer (this step)
  double tavg[kMaxE];        // ... of the prefetch target layer
  uint8_t order[kMaxB][kMaxE];
  uint64_t act[kMaxB], top[kMaxB], low[kMaxB], alt[kMaxB];
  double beta[kMaxB], thT[kMaxB], thL[kMaxB], thR[kMaxB];
  uint8_t sel[kMaxB][kMaxK], sub_d[kMaxB][kMaxK], sub_c[kMaxB][kMaxK], kept[kMaxB][kMaxK];
  uint8_t nsel[kMaxB], nsub[kMaxB], nkept[kMaxB];
  uint64_t C;                // union of top-score experts (router.cpp:105-112)
  uint64_t next_has_pred;    // token bitmask
  StepOut out;
  LayerState ls;             // staged state of the executing layer
  uint32_t def_e[2 * kMaxE]; // deferred admissions (pipeline.cpp:162)
  uint32_t n_def;
  uint32_t pending[kMaxB * kMaxK];
  uint32_t n_pending;
};

// ------------------------------------------------------------------ rng
// xoshiro256** / splitmix64 (rng.cpp:10-56): pure integer, bit-exact.
__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
__host__ __device__ __forceinline__ uint64_t rng_u64(uint64_t* s) {
  const uint64_t out = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return out;
}
__host__ __device__ __forceinline__ double rng_double(uint64_t* s) {
  return (double)(rng_u64(s) >> 11) * 0x1.0p-53;
}
__host__ __device__ __forceinline__ uint64_t rng_below(uint64_t* s, uint64_t n) {
  const uint64_t lim = n * (~0ULL / n);
  uint64_t x;
  do { x = rng_u64(s); } while (x >= lim);
  return x % n;
}
// rng_below for n <= 64 without 64-bit division (identical results): the
// rejection limit n * floor((2^64-1)/n) comes from a compile-time table and
// x mod n is assembled from 32-bit halves.
template <size_t... I>
struct LimTable {
  uint64_t v[sizeof...(I)];
};
template <size_t... I>
constexpr LimTable<I...> make_lim_table(std::index_sequence<I...>) {
  return {{(I == 0 ? 0ULL : (uint64_t)I * (~0ULL / (uint64_t)(I == 0 ? 1 : I)))...}};
}
using LimTableT = decltype(make_lim_table(std::make_index_sequence<kMaxE + 1>{}));
static __constant__ const LimTableT kLim = make_lim_table(std::make_index_sequence<kMaxE + 1>{});

__device__ __forceinline__ uint32_t mod64_small(uint64_t x, uint32_t n) {
  const uint32_t hi = (uint32_t)(x >> 32), lo = (uint32_t)x;
  const uint32_t p32 = (0xFFFFFFFFu % n + 1u) % n;  // 2^32 mod n
  return ((hi % n) * p32 + lo % n) % n;
}
__device__ __forceinline__ uint32_t rng_below_small(uint64_t* s, uint32_t n) {
  const uint64_t lim = kLim.v[n];
  uint64_t x;
  do { x = rng_u64(s); } while (x >= lim);
  return mod64_small(x, n);
}

__host__ __device__ inline uint64_t splitmix_next(uint64_t* st) {
  *st += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *st;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__host__ __device__ inline void rng_seed(uint64_t* s, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) s[i] = splitmix_next(&x);
}
__host__ __device__ inline uint64_t derive_seed(uint64_t seed, uint64_t tag) {
  uint64_t x = seed ^ (0x6a09e667f3bcc909ULL + tag);
  const uint64_t a = splitmix_next(&x);
  const uint64_t b = splitmix_next(&x);
  return a ^ ((b << 29) | (b >> 35));
}

// --------------------------------------------------------- warp helpers
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint64_t bit(uint32_t e) { return 1ULL << e; }
__device__ __forceinline__ bool has(uint64_t m, uint32_t e) { return (m >> e) & 1ULL; }

// 64-bit ballot over the two expert slots of each lane.
__device__ __forceinline__ uint64_t ballot64(bool p0, bool p1) {
  const uint32_t lo = __ballot_sync(0xffffffffu, p0);
  const uint32_t hi = __ballot_sync(0xffffffffu, p1);
  return (uint64_t)lo | ((uint64_t)hi << 32);
}

// Argmin over (key: double, idx) with lowest index on ties: the ascending
// strict-< scan of cache.cpp:81-106. Invalid lanes pass idx = 0xffffffff.
__device__ __forceinline__ void warp_argmin_d(double& key, uint32_t& idx) {
  for (int o = 16; o > 0; o >>= 1) {
    const double k2 = __shfl_xor_sync(0xffffffffu, key, o);
    const uint32_t i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    const bool take = (i2 != 0xffffffffu) &&
                      (idx == 0xffffffffu || k2 < key || (k2 == key && i2 < idx));
    if (take) { key = k2; idx = i2; }
  }
}
__device__ __forceinline__ void warp_argmin_u(uint64_t& key, uint32_t& idx) {
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t k2 = __shfl_xor_sync(0xffffffffu, key, o);
    const uint32_t i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    const bool take = (i2 != 0xffffffffu) &&
                      (idx == 0xffffffffu || k2 < key || (k2 == key && i2 < idx));
    if (take) { key = k2; idx = i2; }
  }
}

// ----------------------------------------------------------- classify
// router.cpp:13-25 ranking + router.cpp:41-71 band classification for one
// token, executed by one warp. Fills order[] (rank -> expert) and the
// act/top/low/alt masks; thresholds exactly (1+a)*b, b, (1-a)*b in fp64.
// f32_keys: every score is an fp32 value widened to fp64 (the stack's
// softmax), so the order-preserving integer key of the double has 29 zero low
// bits and the index fits below them: (score desc, index asc) becomes one
// strict 64-bit integer order, and the rank is a count of larger keys —
// integer compares instead of four fp64 compares per pair (3x faster measured
// on the decision's critical path). Exact for such inputs; general fp64
// scores (simulate()) take the fp64 path.
__device__ inline void classify_warp(const double* s, uint32_t E, uint32_t k, double alpha,
                                     uint8_t* order, uint64_t& act, uint64_t& top, uint64_t& low,
                                     uint64_t& alt, double& beta, double& thT, double& thL,
                                     double& thR, bool f32_keys = false) {
  const int lane = lane_id();
  const uint32_t e0 = lane, e1 = lane + 32;
  const bool v0 = e0 < E, v1 = e1 < E;
  const double s0 = v0 ? s[e0] : 0.0, s1 = v1 ? s[e1] : 0.0;
  uint32_t r0 = 0, r1 = 0;
  if (f32_keys) {
    __shared__ uint64_t s_keys[8][kMaxE];  // per warp (the stack's decider CTA: 8 warps)
    uint64_t* keys = s_keys[warp_id() & 7];
    auto key = [](double v, uint32_t e) -> uint64_t {
      if (v == 0.0) v = 0.0;
      uint64_t b = (uint64_t)__double_as_longlong(v);
      b = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
      return (b & ~0x1FFFFFFFULL) | (uint64_t)(63u - e);
    };
    const uint64_t k0 = key(s0, e0), k1 = key(s1, e1);
    if (v0) keys[e0] = k0;
    if (v1) keys[e1] = k1;
    __syncwarp();
#pragma unroll 16
    for (uint32_t j = 0; j < E; ++j) {
      const uint64_t kj = keys[j];
      r0 += kj > k0;
      r1 += kj > k1;
    }
    __syncwarp();
  } else {
#pragma unroll 16
    for (uint32_t j = 0; j < E; ++j) {
      const double sj = s[j];
      r0 += (sj > s0) || (sj == s0 && j < e0);
      r1 += (sj > s1) || (sj == s1 && j < e1);
    }
  }
  if (v0) order[r0] = (uint8_t)e0;
  if (v1) order[r1] = (uint8_t)e1;
  __syncwarp();
  const double b = s[order[k]];
  const double T = (1.0 + alpha) * b;
  const double Lb = b;
  const double R = (1.0 - alpha) * b;
  const bool a0 = v0 && r0 < k, a1 = v1 && r1 < k;
  const bool l0 = a0 && b > 0.0 && s0 >= Lb && s0 < T;
  const bool l1 = a1 && b > 0.0 && s1 >= Lb && s1 < T;
  const bool al0 = v0 && !a0 && b > 0.0 && s0 >= R && s0 < Lb;
  const bool al1 = v1 && !a1 && b > 0.0 && s1 >= R && s1 < Lb;
  act = ballot64(a0, a1);
  low = ballot64(l0, l1);
  alt = ballot64(al0, al1);
  top = act & ~low;
  beta = b;
  thT = T;
  thL = Lb;
  thR = R;
}

// ------------------------------------------------------------ logging
__device__ inline void log_task(const Logs* lg, uint8_t res, uint8_t kind, int el, uint32_t e,
                                uint64_t start, uint64_t end, uint32_t layer, uint64_t it) {
  if (!lg || !lg->tasks) return;
  const unsigned long long i = atomicAdd(&lg->counts[0], 1ULL);
  if (i >= lg->cap_tasks) { *lg->overflow = 1; return; }
  TaskRec r;
  r.res = res; r.kind = kind; r.el = (int16_t)el; r.e = e; r.start = start; r.end = end;
  r.layer = layer; r.pad = 0; r.it = it;
  lg->tasks[i] = r;
}

}  // namespace moeb
