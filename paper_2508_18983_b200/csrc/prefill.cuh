// prefill.cuh — the prompt (prefill) pass of the MoE stack: N tokens per
// layer, every token routed by plain top-k (the paper's prefill uses the
// traditional offloading path — PAPER.md:358-362 — no substitution: expert
// activation is dense), experts computed as a grouped GEMM
// on the 5th-generation tensor cores.
//
// Per layer, five launches on the stack's stream:
//   pf_router_kernel   RMSNorm (the decode gate's arithmetic) + router logits
//                      on mma.sync (16 tokens x 16 experts per CTA, K split
//                      over warps); writes the shared expert's operand rows
//   pf_topk_kernel     softmax + top-k by counting (score desc, index asc:
//                      plain_top_k, router.cpp:252-260) + combine weights +
//                      the expert histogram (shared-memory, then one global
//                      atomic per expert per CTA); its last CTA builds the
//                      plan with one warp: expert segments (each padded to 16
//                      rows), the item table and the GEMM's unit numbering
//   pf_scatter_kernel  token -> expert permutation (north_star item 4): a
//                      warp's entries of one expert (__match_any_sync) take
//                      consecutive slot rows with one atomic, then the warp
//                      copies each entry's activation row into its slot in the
//                      SW128 K-major operand layout the MMA reads
//   pf_gemm_kernel     grouped SwiGLU: persistent, one CTA per SM; units
//                      gate_up (item, 128 intermediate rows, token tile <= 128)
//                      and down (item, 128 output rows, token tile), token
//                      tiles innermost so a weight tile's re-reads hit L2,
//                      grabbed from one grid counter; tcgen05.mma M = 128,
//                      N = token tile, fp32 accumulators in TMEM (two buffers
//                      of 256 columns), operands staged by cp.async.bulk
//                      (weights are UMMA-tiled, weights.cuh); h = silu(g) * up
//                      kept as bf16 hi + lo (h = hi + lo to 2^-17), both
//                      accumulated by the down MMA; the down epilogue writes
//                      w_slot * y per slot row
//   pf_combine_kernel  per token: shared expert row + its k slot rows in rank
//                      order, residual, bf16 hidden for the next layer
//
// Token slot positions inside an expert segment come from atomics (not
// deterministic), but every GEMM column is an independent dot product and
// the combine sums a token's slots in rank order, so the hidden output is
// bitwise reproducible.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "ffn_umma.cuh"

namespace moeb {

constexpr uint32_t kPfStageBytes = 3 * kUmBlk;  // gate_up: gate + up + x tile; down: down + hi + lo tiles
constexpr uint32_t kPfStages = 4;
constexpr uint32_t kPfThreads = 6 * 32;
constexpr uint32_t kPfTmemCols = 512;           // two buffers x (gate 128 | up 128) columns
constexpr uint32_t kPfNt = 128;                 // token rows per unit (max MMA N of one accumulator pair)
constexpr uint32_t kPfRouterTok = 16;           // tokens per router CTA (one m16 tile)
constexpr uint32_t kPfMaxK = 16;

struct PfItem {
  const unsigned char* w;  // expert weights, UMMA-tiled (weights.cuh)
  uint32_t F;              // intermediate rows (multiple of 128)
  uint32_t row0;           // first slot row (multiple of 16)
  uint32_t n;              // tokens
  uint32_t ntile;          // token tiles (of kPfNt)
  uint32_t tile0;          // first token tile (global index: arrival counters)
  uint32_t gu0, dn0;       // first gate_up / down unit
  uint32_t expert;         // routed expert id, or 0xFFFF for the shared expert
};
struct PfHdr {
  uint32_t n_items, n_gu, n_dn, rows, tiles;
};

// ------------------------------------------------------------ router
struct PfRouterArgs {
  const uint16_t* x;    // [N][d] bf16 layer input
  const uint16_t* wg;   // [E][d] router weights
  const uint16_t* wsg;  // [d] shared-expert gate row (Qwen) or null
  uint16_t* u;          // [N][d] normalised input (bf16)
  unsigned char* xg;    // SW128 activations: rows [0, N) = the shared expert's (null: no shared expert)
  float* logits;        // [N][E + 1]; column E = shared-gate logit
  uint32_t N, d, E, R;
};

// grid (ceil(N / 16), ceil(E / 16)), 256 threads; dynamic smem [16][d + 8]
// bf16. Each CTA: RMSNorm of its 16 tokens (the decode gate's arithmetic,
// layer.cuh gate_phase), then logits of 16 experts on mma.sync m16n8k16:
// warp w takes the K eighth w; the eighths are summed in a fixed order
// (fp32 accumulation).
// Programmatic dependent launch between the per-layer prefill kernels: each
// waits for its predecessor grid (complete, memory visible) before touching
// anything, and lets its own dependent start launching at once, so the
// launch and CTA rasterisation of the next kernel overlap this one's tail.
__device__ __forceinline__ void pf_pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
}

__global__ void __launch_bounds__(256) pf_router_kernel(const __grid_constant__ PfRouterArgs a) {
  pf_pdl_entry();
  extern __shared__ __align__(16) unsigned char pf_rsm[];
  const uint32_t d = a.d, E = a.E, ld = d + 8;
  uint16_t* us = reinterpret_cast<uint16_t*>(pf_rsm);
  __shared__ float inv_rms[kPfRouterTok];
  __shared__ float part[8][kPfRouterTok][16];
  const int lane = lane_id(), warp = warp_id();
  const uint32_t t0 = blockIdx.x * kPfRouterTok, e0 = blockIdx.y * 16;
  const uint32_t nt = min(kPfRouterTok, a.N - t0), nvec = d / 8;
  const bool first = blockIdx.y == 0;
  // router B fragments (Wg rows e0 + lane/4 and e0 + 8 + lane/4, k pairs
  // 2 (lane % 4) and + 8) of 8 k-steps of this warp's K eighth; the first
  // chunk is in flight while x is staged and normalised
  const uint32_t ea = e0 + (lane >> 2), eb = e0 + 8 + (lane >> 2);
  const uint32_t* w0 = ea < E ? reinterpret_cast<const uint32_t*>(a.wg + (size_t)ea * d) + (lane & 3) : nullptr;
  const uint32_t* w1 = eb < E ? reinterpret_cast<const uint32_t*>(a.wg + (size_t)eb * d) + (lane & 3) : nullptr;
  const uint32_t kend_w = (warp + 1) * (d / 8);
  auto load_b = [&](uint32_t c0, uint32_t (&b)[8][4]) {
#pragma unroll
    for (uint32_t i = 0; i < 8; ++i) {
      const uint32_t k0 = c0 + 16 * i, kw = k0 / 2;
      const bool in = k0 < kend_w;
      b[i][0] = in && w0 ? __ldg(w0 + kw) : 0u;
      b[i][1] = in && w0 ? __ldg(w0 + kw + 4) : 0u;
      b[i][2] = in && w1 ? __ldg(w1 + kw) : 0u;
      b[i][3] = in && w1 ? __ldg(w1 + kw + 4) : 0u;
    }
  };
  uint32_t bfr[8][4];
  load_b(warp * (d / 8), bfr);
  for (uint32_t i0 = threadIdx.x; i0 < kPfRouterTok * nvec; i0 += 8 * blockDim.x) {
    uint4 v[8];  // 8 independent 16 B loads in flight per thread
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
      const uint32_t i = i0 + j * blockDim.x, t = i / nvec, c = i % nvec;
      v[j] = i < kPfRouterTok * nvec && t < nt ? __ldg(reinterpret_cast<const uint4*>(a.x + (size_t)(t0 + t) * d) + c)
                                               : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
      const uint32_t i = i0 + j * blockDim.x, t = i / nvec, c = i % nvec;
      if (i < kPfRouterTok * nvec) *reinterpret_cast<uint4*>(us + (size_t)t * ld + c * 8) = v[j];
    }
  }
  __syncthreads();
  for (uint32_t t = warp; t < kPfRouterTok; t += 8) {
    float ss = 0.f;
    for (uint32_t c = lane; c < nvec; c += 32) {
      const uint4 v = *reinterpret_cast<const uint4*>(us + (size_t)t * ld + c * 8);
      ss += dot8(v, v);
    }
    ss = warp_sum(ss);
    if (lane == 0) inv_rms[t] = __frsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)d), 1e-6f));
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kPfRouterTok * nvec; i += blockDim.x) {
    const uint32_t t = i / nvec, c = i % nvec;
    uint4* p = reinterpret_cast<uint4*>(us + (size_t)t * ld + c * 8);
    const uint4 v = *p;
    const float r = inv_rms[t];
    const uint32_t in[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float lo = __fmul_rn(__uint_as_float(in[j] << 16), r);
      const float hi = __fmul_rn(__uint_as_float(in[j] & 0xffff0000u), r);
      o[j] = (uint32_t)f32_to_bf16_rne(lo) | ((uint32_t)f32_to_bf16_rne(hi) << 16);
    }
    const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
    *p = ov;
    if (first && t < nt) {
      reinterpret_cast<uint4*>(a.u + (size_t)(t0 + t) * d)[c] = ov;
      if (a.xg) {  // the shared expert's operand rows = the tokens in order
        const uint32_t r = t0 + t;
        const size_t off = (size_t)(c >> 3) * a.R * 128u + (r >> 3) * 1024u + (r & 7u) * 128u + (((c ^ r) & 7u) << 4);
        *reinterpret_cast<uint4*>(a.xg + off) = ov;
      }
    }
  }
  __syncthreads();
  {
    const uint32_t kq = warp, kspan = d / 8, k_beg = kq * kspan, k_end = k_beg + kspan;
    float acc[2][4] = {};
    const uint32_t a_addr = smem_u32(us + (size_t)(lane & 15) * ld + (lane >> 4) * 8);
    // chunks of 8 k-steps: the B fragments of the next chunk are loaded while
    // this one's MMAs run (the first chunk was loaded before the RMSNorm)
    uint32_t bn[8][4];
    for (uint32_t c0 = k_beg; c0 < k_end; c0 += 128) {
      uint32_t bc[8][4];
#pragma unroll
      for (uint32_t i = 0; i < 8; ++i)
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) bc[i][q] = c0 == k_beg ? bfr[i][q] : bn[i][q];
      if (c0 + 128 < k_end) load_b(c0 + 128, bn);
#pragma unroll
      for (uint32_t i = 0; i < 8; ++i) {
        const uint32_t k0 = c0 + 16 * i;
        if (k0 < k_end) {
          uint32_t af[4];
          ldsm_x4(a_addr + k0 * 2, af);
          mma16816(acc[0], af, bc[i][0], bc[i][1]);
          mma16816(acc[1], af, bc[i][2], bc[i][3]);
        }
      }
    }
#pragma unroll
    for (uint32_t j = 0; j < 2; ++j) {
      const uint32_t r = lane >> 2, e = 8 * j + 2 * (lane & 3);
      part[kq][r][e] = acc[j][0];
      part[kq][r][e + 1] = acc[j][1];
      part[kq][r + 8][e] = acc[j][2];
      part[kq][r + 8][e + 1] = acc[j][3];
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kPfRouterTok * 16; i += blockDim.x) {
    const uint32_t t = i / 16, e = i % 16;
    if (t < nt && e0 + e < E) {
      float v = 0.f;
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q) v += part[q][t][e];  // fixed order
      a.logits[(size_t)(t0 + t) * (E + 1) + e0 + e] = v;
    }
  }
  if (first && a.wsg)  // Qwen shared-expert gate logit
    for (uint32_t t = warp; t < nt; t += 8) {
      float s = 0.f;
      const uint4* wv = reinterpret_cast<const uint4*>(a.wsg);
      for (uint32_t c = lane; c < nvec; c += 32)
        s += dot8(__ldg(wv + c), *reinterpret_cast<const uint4*>(us + (size_t)t * ld + c * 8));
      s = warp_sum(s);
      if (lane == 0) a.logits[(size_t)(t0 + t) * (E + 1) + E] = s;
    }
}

// ------------------------------------------------------------ plan
struct PfPlanArgs {
  uint32_t* cnt;         // [E] tokens per expert (re-zeroed here for the next layer)
  uint32_t* cursor;      // [E] next free slot row of each expert segment
  const LayerState* ls;  // this layer's cache state (residency, slots)
  const unsigned char* slot_base;   // this layer's cache slots
  const unsigned char* stage_base;  // staging of the non-resident experts (by expert id)
  const unsigned char* shared_w;    // shared expert (null: none)
  const unsigned char* tiled_base;  // non-null: every routed expert re-tiled here (by expert id)
  uint64_t expert_bytes;
  uint32_t N, E, d, F, S;
  PfItem* items;
  PfHdr* hdr;
};

// One warp: the expert segments (each padded to 16 rows, experts in
// ascending order after the shared expert's N rows), the item table and the
// GEMM's unit numbering (lane-parallel prefix sums).
__device__ void pf_plan_warp(const PfPlanArgs& a) {
  const int lane = lane_id();
  const uint32_t nmt = a.d / 128, ftl = a.F / 128;
  uint32_t rows = 0, tiles = 0, gu = 0, n_items = 0;
  if (a.S) {
    PfItem it{};
    it.w = a.shared_w;
    it.F = a.S;
    it.n = a.N;
    it.ntile = (a.N + kPfNt - 1) / kPfNt;
    it.expert = 0xFFFFu;
    if (lane == 0) a.items[0] = it;
    rows = (a.N + 15) & ~15u;
    tiles = it.ntile;
    gu = it.ntile * (a.S / 128);
    n_items = 1;
  }
  const uint64_t mask = a.ls->mask;
  for (uint32_t e0 = 0; e0 < a.E; e0 += 32) {
    const uint32_t e = e0 + lane;
    const uint32_t c = e < a.E ? __ldcg(&a.cnt[e]) : 0u;
    const uint32_t pr = (c + 15) & ~15u, nt = (c + kPfNt - 1) / kPfNt;
    uint32_t sr = pr, st = nt, sg = nt * ftl, si = c ? 1u : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t vr = __shfl_up_sync(0xffffffffu, sr, o), vt = __shfl_up_sync(0xffffffffu, st, o);
      const uint32_t vg = __shfl_up_sync(0xffffffffu, sg, o), vi = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) { sr += vr; st += vt; sg += vg; si += vi; }
    }
    if (c) {
      PfItem it{};
      const bool res = (mask >> e) & 1ull;
      it.w = a.tiled_base ? a.tiled_base + (uint64_t)e * a.expert_bytes
             : res        ? a.slot_base + (uint64_t)a.ls->slot_of[e] * a.expert_bytes
                          : a.stage_base + (uint64_t)e * a.expert_bytes;
      it.F = a.F;
      it.row0 = rows + sr - pr;
      it.n = c;
      it.ntile = nt;
      it.tile0 = tiles + st - nt;
      it.gu0 = gu + sg - nt * ftl;
      it.expert = e;
      a.items[n_items + si - 1] = it;
    }
    if (e < a.E) {
      a.cursor[e] = rows + sr - pr;
      a.cnt[e] = 0;
    }
    rows += __shfl_sync(0xffffffffu, sr, 31);
    tiles += __shfl_sync(0xffffffffu, st, 31);
    gu += __shfl_sync(0xffffffffu, sg, 31);
    n_items += __shfl_sync(0xffffffffu, si, 31);
  }
  __syncwarp();
  uint32_t dn = gu;  // down units after every gate_up unit, in item order
  for (uint32_t i0 = 0; i0 < n_items; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t v = i < n_items ? __ldcg(&a.items[i].ntile) * nmt : 0u;
    uint32_t s = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    if (i < n_items) a.items[i].dn0 = dn + s - v;
    dn += __shfl_sync(0xffffffffu, s, 31);
  }
  if (lane == 0) *a.hdr = PfHdr{n_items, gu, dn - gu, rows, tiles};
}

// ------------------------------------------------------------ top-k
struct PfTopkArgs {
  const float* logits;   // [N][E + 1]
  float* scores;         // [N][E] fp32 softmax scores
  uint8_t* sel;          // [N][k] selected experts in rank order
  float* wts;            // [N][k] combine weights
  float* slot_w;         // [R]: rows [0, N) = the shared expert's weight per token (null: no shared expert)
  uint32_t* cnt;         // [E] tokens per expert (histogram; zero on entry)
  uint32_t* ticket;      // CTAs done (the last one builds the plan; reset to 0)
  PfPlanArgs plan;
  uint32_t N, E, k;
  int32_t renormalize, shared_gate;
  float routed_scale;
};

// One warp per token: softmax, rank by counting (score desc, index asc:
// plain_top_k, router.cpp:252-260), combine weights; the expert histogram is
// aggregated per CTA in shared memory, one global atomic per expert per CTA;
// the last CTA to finish builds the plan (pf_plan_warp).
__global__ void __launch_bounds__(256) pf_topk_kernel(const __grid_constant__ PfTopkArgs a) {
  pf_pdl_entry();
  __shared__ uint32_t hist[kMaxE];
  const int lane = lane_id();
  const uint32_t E = a.E, k = a.k;
  for (uint32_t e = threadIdx.x; e < kMaxE; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const uint32_t t = blockIdx.x * 8 + warp_id();
  if (t < a.N) {
    const float* lg = a.logits + (size_t)t * (E + 1);
    float sc[2];
    {
      const float l0 = (uint32_t)lane < E ? lg[lane] : -INFINITY;
      const float l1 = (uint32_t)lane + 32 < E ? lg[lane + 32] : -INFINITY;
      float m = fmaxf(l0, l1);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      const float x0 = (uint32_t)lane < E ? expf(l0 - m) : 0.f;
      const float x1 = (uint32_t)lane + 32 < E ? expf(l1 - m) : 0.f;
      float s = x0 + x1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      sc[0] = __fdiv_rn(x0, s);
      sc[1] = __fdiv_rn(x1, s);
    }
    if ((uint32_t)lane < E) a.scores[(size_t)t * E + lane] = sc[0];
    if ((uint32_t)lane + 32 < E) a.scores[(size_t)t * E + lane + 32] = sc[1];
    uint32_t rk[2] = {0u, 0u};
    for (uint32_t j = 0; j < E; ++j) {
      const float sj = __shfl_sync(0xffffffffu, sc[j >> 5], j & 31);
#pragma unroll
      for (uint32_t h = 0; h < 2; ++h) {
        const uint32_t e = lane + 32 * h;
        rk[h] += (sj > sc[h] || (sj == sc[h] && j < e)) ? 1u : 0u;
      }
    }
    const bool s0 = (uint32_t)lane < E && rk[0] < k, s1 = (uint32_t)lane + 32 < E && rk[1] < k;
    float den = 1.f;
    if (a.renormalize) {  // selected scores summed in rank order
      den = 0.f;
      for (uint32_t r = 0; r < k; ++r) {
        const uint32_t hit = __ballot_sync(0xffffffffu, (s0 && rk[0] == r) || (s1 && rk[1] == r));
        den += __shfl_sync(0xffffffffu, (s0 && rk[0] == r) ? sc[0] : sc[1], __ffs(hit) - 1);
      }
    }
#pragma unroll
    for (uint32_t h = 0; h < 2; ++h) {
      if (h ? s1 : s0) {
        const uint32_t e = lane + 32 * h;
        a.sel[(size_t)t * k + rk[h]] = (uint8_t)e;
        float w = sc[h];
        if (a.renormalize) w = __fdiv_rn(w, den);
        a.wts[(size_t)t * k + rk[h]] = __fmul_rn(w, a.routed_scale);
        atomicAdd(&hist[e], 1u);
      }
    }
    if (a.slot_w && lane == 0) a.slot_w[t] = a.shared_gate ? 1.f / (1.f + expf(-lg[E])) : 1.f;
  }
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < E; e += blockDim.x)
    if (hist[e]) atomicAdd(&a.cnt[e], hist[e]);
  __shared__ uint32_t s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    pf_plan_warp(a.plan);
    if (threadIdx.x == 0) *a.ticket = 0;
  }
}

// ------------------------------------------------------------ scatter
// The token -> expert permutation: a CTA takes 32 (token, rank) entries;
// warp 0 gives the entries of one expert (__match_any_sync) consecutive slot
// rows with one atomic on the expert's cursor; then the 8 warps copy the
// entries' activation rows into their slots (SW128: 16 B chunk c of row r in
// K-block c / 8 at chunk position (c ^ r) % 8).
struct PfScatterArgs {
  const uint8_t* sel;    // [N][k]
  const float* wts;      // [N][k]
  const uint16_t* u;     // [N][d]
  uint32_t* cursor;      // [E]
  float* slot_w;         // [R]
  int32_t* entry_slot;   // [N][k]
  unsigned char* xg;     // [d/64][R][128 B]
  uint32_t N, k, d, R;
  uint32_t* ctr_zero;    // the GEMM's unit / tile counters, zeroed here (the previous GEMM is complete)
  uint32_t n_ctr;
};

__global__ void __launch_bounds__(256) pf_scatter_kernel(const __grid_constant__ PfScatterArgs a) {
  pf_pdl_entry();
  __shared__ uint32_t s_slot[32];
  const int lane = lane_id(), warp = warp_id();
  const uint32_t n = a.N * a.k, nvec = a.d / 8;
  if (blockIdx.x == 0)
    for (uint32_t i = threadIdx.x; i < a.n_ctr; i += blockDim.x) a.ctr_zero[i] = 0;
  const uint32_t i0 = blockIdx.x * 32;
  if (warp == 0) {
    const uint32_t i = i0 + lane;
    const bool live = i < n;
    const uint32_t e = live ? a.sel[i] : 0xFFu;
    const uint32_t act = __ballot_sync(0xffffffffu, live);
    if (live) {
      const uint32_t peers = __match_any_sync(act, e);
      const int leader = __ffs(peers) - 1;
      uint32_t b = 0;
      if (lane == leader) b = atomicAdd(&a.cursor[e], __popc(peers));
      b = __shfl_sync(peers, b, leader);
      const uint32_t slot = b + __popc(peers & ((1u << lane) - 1u));
      a.slot_w[slot] = a.wts[i];
      a.entry_slot[i] = (int32_t)slot;
      s_slot[lane] = slot;
    }
  }
  __syncthreads();
  for (uint32_t j = warp; j < 32 && i0 + j < n; j += 8) {
    const uint32_t r = s_slot[j];
    const uint4* src = reinterpret_cast<const uint4*>(a.u + (size_t)((i0 + j) / a.k) * a.d);
    for (uint32_t c0 = lane; c0 < nvec; c0 += 8 * 32) {
      uint4 v[8];  // 8 independent loads in flight per lane
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q)
        if (c0 + q * 32 < nvec) v[q] = __ldg(src + c0 + q * 32);
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q) {
        const uint32_t c = c0 + q * 32;
        if (c < nvec) {
          const size_t off = (size_t)(c >> 3) * a.R * 128u + (r >> 3) * 1024u + (r & 7u) * 128u + (((c ^ r) & 7u) << 4);
          *reinterpret_cast<uint4*>(a.xg + off) = v[q];
        }
      }
    }
  }
}

// ------------------------------------------------------------ re-tiling
// Batch-1 stacks keep experts row-interleaved ([F][3][d], the split-K GEMV's
// layout); prefill re-tiles each layer's experts into the UMMA layout
// (weights.cuh tiled_coords) through HBM first. One CTA per 16 KB tile:
// gate / up tiles are row copies with the SW128 chunk swizzle; down tiles
// (128 outputs x 64 intermediate rows, K = intermediate) are transposed
// through shared memory. blockIdx.y = expert (gridDim.y - 1 = the shared
// expert when shared_src is set); a routed expert's source is its cache slot
// when resident, else the staging area.
struct PfRetileArgs {
  const LayerState* ls;
  const unsigned char* slot_base;
  const unsigned char* stage_base;
  const unsigned char* shared_src;  // shared expert (rows layout) or null
  unsigned char* dst;               // [E][expert_bytes] then the shared expert
  uint64_t expert_bytes;
  uint32_t E, d, F, S;
};

__global__ void __launch_bounds__(256) pf_retile_kernel(const __grid_constant__ PfRetileArgs a) {
  pf_pdl_entry();
  __shared__ __align__(16) uint16_t tr[64][128 + 8];
  const uint32_t e = blockIdx.y, d = a.d;
  const bool sh = a.shared_src && e == a.E;
  const uint32_t F = sh ? a.S : a.F;
  const uint32_t n_gu = (F / 128) * (d / 64) * 2, n_dn = (d / 128) * (F / 64);
  if (blockIdx.x >= n_gu + n_dn) return;
  const unsigned char* src;
  if (sh) {
    src = a.shared_src;
  } else {
    const bool res = (a.ls->mask >> e) & 1ull;
    src = res ? a.slot_base + (uint64_t)a.ls->slot_of[e] * a.expert_bytes : a.stage_base + (uint64_t)e * a.expert_bytes;
  }
  const uint16_t* w = reinterpret_cast<const uint16_t*>(src);
  unsigned char* dst = a.dst + (uint64_t)e * a.expert_bytes + (uint64_t)blockIdx.x * kUmBlk;
  if (blockIdx.x < n_gu) {
    // gate_up tile (unit u, K-block kb, gate|up): out row rr = F-row u*128 + rr
    const uint32_t t = blockIdx.x, which = t & 1, kb = (t >> 1) % (d / 64), u = (t >> 1) / (d / 64);
    for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) {
      const uint32_t rr = i >> 3, j = i & 7;
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(w + (size_t)(u * 128 + rr) * 3 * d + which * d + kb * 64 + 8 * j));
      *reinterpret_cast<uint4*>(dst + sw128_off(rr, 8 * j)) = v;
    }
  } else {
    // down tile (output unit mt, K-block kb): element (m, r) = down column r, entry m
    const uint32_t t = blockIdx.x - n_gu, kb = t % (F / 64), mt = t / (F / 64);
    for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) {
      const uint32_t r = i >> 4, j = i & 15;
      *reinterpret_cast<uint4*>(&tr[r][8 * j]) =
          __ldg(reinterpret_cast<const uint4*>(w + (size_t)(kb * 64 + r) * 3 * d + 2 * d + mt * 128 + 8 * j));
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) {
      const uint32_t m = i >> 3, j = i & 7;
      uint32_t o[4];
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q) o[q] = (uint32_t)tr[8 * j + 2 * q][m] | ((uint32_t)tr[8 * j + 2 * q + 1][m] << 16);
      *reinterpret_cast<uint4*>(dst + sw128_off(m, 8 * j)) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// ------------------------------------------------------------ grouped GEMM
struct PfGemmArgs {
  const PfItem* items;
  const PfHdr* hdr;
  const unsigned char* xg;  // [d/64][R][128 B] activations (SW128)
  unsigned char* hg;        // [Fmax/64][2][R][128 B] h hi / lo (SW128)
  float* out;               // [R][d] w_slot * expert output
  const float* slot_w;      // [R]
  uint32_t* ctr;            // [0] unit grab, [1] CTAs done, [2 + tile] gate_up arrivals
  uint32_t d, R;
};

struct PfRec {
  uint32_t kind;  // 0 gate_up, 1 down, 2 end
  uint32_t item, tile, idx, nt, nrows;
};

__global__ void __launch_bounds__(kPfThreads, 1) pf_gemm_kernel(const __grid_constant__ PfGemmArgs a) {
  pf_pdl_entry();
  extern __shared__ unsigned char pf_smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kPfStages], empty_bar[kPfStages];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t rfull_bar[kUmRec], rempty_bar[kUmRec];
  __shared__ PfRec recs[kUmRec];
  __shared__ PfItem s_items[kMaxItems];
  __shared__ uint32_t s_tmem;
  const int warp = warp_id(), lane = lane_id();
  const uint32_t d = a.d, R = a.R, nkb = d / 64, nmt = d / 128;
  const uint32_t raw_addr = smem_u32(pf_smem_raw);
  unsigned char* ring = pf_smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  const uint32_t ring_addr = smem_u32(ring);
  const PfHdr hdr = *a.hdr;
  for (uint32_t i = threadIdx.x; i < hdr.n_items; i += blockDim.x) s_items[i] = a.items[i];
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < kPfStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4);
    }
    for (uint32_t j = 0; j < kUmRec; ++j) {
      mbar_init(&rfull_bar[j], 1);
      mbar_init(&rempty_bar[j], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "n"(kPfTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    um_fence_before();
  }
  __syncthreads();
  um_fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      const uint64_t pol_w = l2_evict_first_policy(), pol_x = l2_evict_last_policy();
      const uint32_t total = hdr.n_gu + hdr.n_dn;
      uint32_t k = 0, u = 0;
      for (uint32_t unit = atomicAdd(&a.ctr[0], 1u); unit < total; unit = atomicAdd(&a.ctr[0], 1u)) {
        PfRec r{};
        const bool gu = unit < hdr.n_gu;
        uint32_t i = 0;
        // the item holding the unit (items are in unit order)
        for (uint32_t j = 1; j < hdr.n_items; ++j)
          if ((gu ? s_items[j].gu0 : s_items[j].dn0) <= unit) i = j;
        const PfItem& it = s_items[i];
        const uint32_t q = unit - (gu ? it.gu0 : it.dn0);
        r.kind = gu ? 0u : 1u;
        r.item = i;
        r.idx = q / it.ntile;  // token tiles innermost: a weight tile's re-reads hit L2
        r.tile = q % it.ntile;
        r.nrows = min(kPfNt, it.n - r.tile * kPfNt);
        r.nt = (r.nrows + 15) & ~15u;
        {
          const uint32_t j = u % kUmRec;
          mbar_wait(&rempty_bar[j], ((u / kUmRec) & 1) ^ 1);
          recs[j] = r;
          mbar_arrive(&rfull_bar[j]);
          ++u;
        }
        const size_t row = (size_t)it.row0 + r.tile * kPfNt;
        const uint32_t xb = r.nt * 128;
        if (gu) {
          const unsigned char* wsrc = it.w + ((size_t)r.idx * nkb) * kUmA;
          for (uint32_t kb = 0; kb < nkb; ++kb, ++k) {
            const uint32_t st = k % kPfStages;
            mbar_wait(&empty_bar[st], ((k / kPfStages) & 1) ^ 1);
            mbar_expect_tx(&full_bar[st], kUmA + xb);
            bulk_g2s(ring + st * kPfStageBytes, wsrc + (size_t)kb * kUmA, kUmA, &full_bar[st], pol_w);
            bulk_g2s(ring + st * kPfStageBytes + kUmA, a.xg + ((size_t)kb * R + row) * 128, xb, &full_bar[st], pol_x);
          }
        } else {
          // h of this (item, token tile): every gate_up unit must have landed
          wait_ctr_ge(&a.ctr[2 + it.tile0 + r.tile], it.F / 128, 10u);
          fence_proxy_async_global();
          const uint32_t nfb = it.F / 64;
          const unsigned char* wsrc = it.w + (size_t)2 * it.F * d * 2 + (size_t)r.idx * nfb * kUmBlk;
          for (uint32_t kb = 0; kb < nfb; ++kb, ++k) {
            const uint32_t st = k % kPfStages;
            mbar_wait(&empty_bar[st], ((k / kPfStages) & 1) ^ 1);
            mbar_expect_tx(&full_bar[st], kUmBlk + 2 * xb);
            unsigned char* dst = ring + st * kPfStageBytes;
            bulk_g2s(dst, wsrc + (size_t)kb * kUmBlk, kUmBlk, &full_bar[st], pol_w);
            bulk_g2s(dst + kUmBlk, a.hg + ((size_t)(2 * kb) * R + row) * 128, xb, &full_bar[st], pol_x);
            bulk_g2s(dst + kUmBlk + xb, a.hg + ((size_t)(2 * kb + 1) * R + row) * 128, xb, &full_bar[st], pol_x);
          }
        }
      }
      const uint32_t j = u % kUmRec;
      mbar_wait(&rempty_bar[j], ((u / kUmRec) & 1) ^ 1);
      recs[j] = PfRec{2u, 0u, 0u, 0u, 0u, 0u};
      mbar_arrive(&rfull_bar[j]);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      uint32_t k = 0;
      for (uint32_t u = 0;; ++u) {
        const uint32_t j = u % kUmRec;
        mbar_wait(&rfull_bar[j], (u / kUmRec) & 1);
        const PfRec r = recs[j];
        if (r.kind == 2) break;
        const uint32_t b = u & 1;
        mbar_wait(&tempty_bar[b], ((u >> 1) & 1) ^ 1);
        um_fence_after();
        const uint32_t acc = tmem + b * 256, idesc = um_idesc(r.nt), xb = r.nt * 128;
        const uint32_t n_st = r.kind == 0 ? nkb : s_items[r.item].F / 64;
        for (uint32_t s = 0; s < n_st; ++s, ++k) {
          const uint32_t st = k % kPfStages;
          mbar_wait(&full_bar[st], (k / kPfStages) & 1);
          um_fence_after();
          const uint32_t sa = ring_addr + st * kPfStageBytes;
          if (r.kind == 0) {
#pragma unroll
            for (uint32_t kk = 0; kk < 4; ++kk) {
              const uint64_t bx = um_desc(sa + kUmA + kk * 32);
              um_mma(acc, um_desc(sa + kk * 32), bx, idesc, (s | kk) != 0);
              um_mma(acc + 128, um_desc(sa + kUmBlk + kk * 32), bx, idesc, (s | kk) != 0);
            }
          } else {
#pragma unroll
            for (uint32_t kk = 0; kk < 4; ++kk) {
              const uint64_t aw = um_desc(sa + kk * 32);
              um_mma(acc, aw, um_desc(sa + kUmBlk + kk * 32), idesc, (s | kk) != 0);
              um_mma(acc, aw, um_desc(sa + kUmBlk + xb + kk * 32), idesc, 1u);
            }
          }
          um_commit(&empty_bar[st]);
        }
        um_commit(&tfull_bar[b]);
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue
    const uint32_t q = warp & 3, et = (warp - 2) * 32 + lane;
    for (uint32_t u = 0;; ++u) {
      const uint32_t j = u % kUmRec;
      mbar_wait(&rfull_bar[j], (u / kUmRec) & 1);
      const PfRec r = recs[j];
      if (r.kind == 2) break;
      const PfItem& it = s_items[r.item];
      const uint32_t b = u & 1;
      mbar_wait(&tfull_bar[b], (u >> 1) & 1);
      um_fence_after();
      const uint32_t ta = tmem + ((q * 32) << 16) + b * 256;
      const uint32_t row0 = it.row0 + r.tile * kPfNt;
      if (r.kind == 0) {
        // intermediate row f of the item -> h K-block f / 64, column f % 64
        const uint32_t f = r.idx * 128 + q * 32 + lane;
        unsigned char* hhi = a.hg + (size_t)(2 * (f >> 6)) * R * 128;
        unsigned char* hlo = hhi + (size_t)R * 128;
        const uint32_t col = f & 63;
        for (uint32_t c0 = 0; c0 < r.nt; c0 += 16) {
          float g[16], up[16];
          um_ld16(ta + c0, g);
          um_ld16(ta + 128 + c0, up);
          um_ld_wait();
#pragma unroll
          for (uint32_t i = 0; i < 16; ++i) {
            const uint32_t c = c0 + i, rr = row0 + c;
            const float h = c < r.nrows ? (g[i] / (1.f + __expf(-g[i]))) * up[i] : 0.f;
            const uint16_t hi = f32_to_bf16_rne(h);
            const uint16_t lo = f32_to_bf16_rne(h - bf2f(hi));
            *reinterpret_cast<uint16_t*>(hhi + sw128_off(rr, col)) = hi;
            *reinterpret_cast<uint16_t*>(hlo + sw128_off(rr, col)) = lo;
          }
        }
        um_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[b]);
        fence_proxy_async_global();  // h is read by the down units' bulk copies
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (et == 0) {
          __threadfence();
          atomicAdd(&a.ctr[2 + it.tile0 + r.tile], 1u);
          mbar_arrive(&rempty_bar[j]);
        }
      } else {
        const uint32_t m = r.idx * 128 + q * 32 + lane;
        for (uint32_t c0 = 0; c0 < r.nt; c0 += 16) {
          float v[16];
          um_ld16(ta + c0, v);
          um_ld_wait();
#pragma unroll
          for (uint32_t i = 0; i < 16; ++i) {
            const uint32_t c = c0 + i;
            if (c < r.nrows) __stcg(a.out + (size_t)(row0 + c) * d + m, v[i] * __ldg(a.slot_w + row0 + c));
          }
        }
        um_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[b]);
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (et == 0) mbar_arrive(&rempty_bar[j]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kPfTmemCols));
}

// ------------------------------------------------------------ combine
// hidden[t] = bf16(x[t] + shared row t + the token's k slot rows in rank order);
// y (nullable) keeps the fp32 layer output. One thread per 4 outputs.
__global__ void __launch_bounds__(256) pf_combine_kernel(const uint16_t* __restrict__ x, const float* __restrict__ out,
                                                         const int32_t* __restrict__ entry_slot, uint16_t* __restrict__ xo,
                                                         float* __restrict__ y, uint32_t N, uint32_t d, uint32_t k,
                                                         uint32_t shared) {
  pf_pdl_entry();
  const uint32_t per = d / 4;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N * per; i += gridDim.x * blockDim.x) {
    const uint32_t t = i / per, c = (i % per) * 4;
    float4 s = shared ? __ldcg(reinterpret_cast<const float4*>(out + (size_t)t * d + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t j = 0; j < k; ++j) {
      const int32_t sl = __ldg(entry_slot + (size_t)t * k + j);
      const float4 v = __ldcg(reinterpret_cast<const float4*>(out + (size_t)sl * d + c));
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    const uint2 xv = *reinterpret_cast<const uint2*>(x + (size_t)t * d + c);
    const float o0 = __uint_as_float(xv.x << 16) + s.x, o1 = __uint_as_float(xv.x & 0xffff0000u) + s.y;
    const float o2 = __uint_as_float(xv.y << 16) + s.z, o3 = __uint_as_float(xv.y & 0xffff0000u) + s.w;
    uint2 ov;
    ov.x = (uint32_t)f32_to_bf16_rne(o0) | ((uint32_t)f32_to_bf16_rne(o1) << 16);
    ov.y = (uint32_t)f32_to_bf16_rne(o2) | ((uint32_t)f32_to_bf16_rne(o3) << 16);
    *reinterpret_cast<uint2*>(xo + (size_t)t * d + c) = ov;
    if (y) *reinterpret_cast<float4*>(y + (size_t)t * d + c) = s;
  }
}

}  // namespace moeb
