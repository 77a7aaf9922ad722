// ffn_tma.cuh — persistent grouped SwiGLU FFN with a bulk-copy (TMA) weight
// pipeline (sm_100a).
//
// One CTA per SM: warp 0 is the producer, warps 1..kConsumers compute. Each
// CTA owns a fixed contiguous share of every item's rows:
//   gate_up : rows [F*c/G, F*(c+1)/G) of W_gate and W_up (h = silu(g)*u)
//   down    : output rows [d*c/G, d*(c+1)/G) of W_down, accumulated over the
//             items in plan order (deterministic, no atomics)
// The producer streams those rows through a ring of 32 KB shared-memory
// stages with cp.async.bulk (one or two contiguous copies per stage,
// completion on an mbarrier transaction count); consumers read rows from
// shared memory. ~200 KB of weights in flight per SM keeps HBM saturated
// without register pressure. Items whose weights are still on the PCIe copy
// stream are gated by the producer on copies_done; the down pass of an item
// waits for every CTA's gate_up rows of that item (per-item grid counter).
// The decode FFN is a GEMV (B <= 32 tokens): memory-bound, no tensor cores.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "layer.cuh"

namespace moeb {

constexpr int kMaxStages = 12;
// FFN grid counters (zeroed by the decide kernel before every launch):
// [0, kMaxItems) per-item gate_up completion (CTAs), then the deferred-copy
// barrier, the exit counter and the dynamic gate_up chunk counter
constexpr int kFfnD2dCtr = kMaxItems;
constexpr int kFfnExitCtr = kMaxItems + 1;
constexpr int kFfnGuCtr = kMaxItems + 2;        // dynamic gate_up chunks, final plan
constexpr int kFfnReadyDoneCtr = kMaxItems + 3;  // CTAs done with the final plan's ready gate_up
constexpr int kFfnSpecGuCtr = kMaxItems + 4;     // dynamic gate_up chunks, speculative plan
constexpr int kFfnSpecDoneCtr = kMaxItems + 5;   // CTAs done with the speculative gate_up
constexpr int kFfnRedCtr = kMaxItems + 6;        // end-of-kernel reduction barrier (split-K kernel)
constexpr int kFfnCtrWords = kMaxItems + 7;
constexpr int kTlWords = 16;  // timeline record words per layer-step
constexpr size_t kPlanSmem = (sizeof(Plan) + 15) & ~(size_t)15;  // plan copy in smem, 16 B aligned

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// Weights are streamed exactly once per decode step: load them with an L2
// evict-first policy so they do not push the small decision state, plan and
// activations out of L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

struct FfnTArgs {
  const Plan* plan;
  const uint16_t* u;       // [B][d]
  const uint16_t* x_in;    // [B][d]
  uint16_t* x_out;         // [B][d]
  float* y_out;            // [B][d]
  uint16_t* x_pred;        // [B][d] or null: bf16(x_in + the shared expert's and resident hits'
                           // contributions) — the partial forward the next layer's predictor reads
  float* h;                // [kMaxItems][B][Fmax]
  uint32_t* ctr;           // [0,kMaxItems) item gate_up done, [kMaxItems] d2d barrier, [kMaxItems+1] exit
  const uint32_t* copies_done;
  uint32_t* ffn_done;
  uint32_t B, d, Fmax, stages;
  uint32_t stage_bytes;    // bytes per ring stage (multiple of 1 KB)
  uint32_t hbuf_bytes;     // smem reserved for staging h of the ready items
  uint32_t acc_rows;       // ceil(d / grid): down rows per CTA
  uint32_t plan_smem;      // bytes of the plan header + items kept in smem
  uint32_t x_smem;         // bytes of the activation copy in smem (0: B == 1, d <= 2048, registers)
  uint32_t dbg;            // microbenchmark knobs: 1 no consumer math, 2 skip down pass
  uint64_t* tstamp;        // microbenchmark: per-CTA phase timestamps [grid][8] (nullable)
  uint64_t* tl;            // timeline trace: this launch's [8] record (nullable): 0 final plan in
                           // hand (CTA 0), 1 CTA 0's producer saw its last upload, 2 end (last
                           // CTA), 6 speculative plan in hand (CTA 0)
  const Plan* spec_plan;   // speculative plan (null: none); published when *spec_flag == seq
  const uint32_t* spec_flag;
  uint32_t seq;
  uint32_t unit_rows;      // split-K kernel: intermediate rows per grid-counter grab (0: default)
  uint32_t deterministic;  // split-K kernel: static row -> (CTA, warp) assignment (bitwise-reproducible sums)
  uint32_t shared_first;   // split-K kernel: item 0 (shared expert) of spec_plan released alone by spec_flag[2]
  const uint16_t* shared_w;  // split-K kernel with shared_first: the layer's shared expert (rows prefetched
  uint32_t shared_F;         //   into the ring before the release), its intermediate rows
  const uint32_t* spec_done;  // split-K kernel: speculative upload generations landed, per buffer [2]
};

// Row range of CTA c out of G over n rows.
__device__ __forceinline__ void share(uint32_t n, uint32_t c, uint32_t G, uint32_t& lo, uint32_t& hi) {
  lo = n * c / G;  // n * G < 2^32 for every shape we accept
  hi = n * (c + 1) / G;
}

// Tile schedule shared by the producer and the consumers: gate_up tiles of
// the ready items, down tiles of the ready items, then per waiting item its
// gate_up tiles followed by its down tiles.
struct TileIter {
  uint32_t phase;      // 0 gu-ready, 1 dn-ready, 2 waiting (gu then dn)
  uint32_t item;
  uint32_t sub;        // 0 gu, 1 dn  (phase 2)
  uint32_t row;        // next row of the current (item, kind)
};

// ---- packed fp32 math (sm_100 FFMA2): two bf16 weights unpacked into an
// f32x2 pair, multiplied with an fp32 pair and accumulated as a pair.
__device__ __forceinline__ unsigned long long f2pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float f2sum(unsigned long long v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return lo + hi;
}
__device__ __forceinline__ void ffma2(unsigned long long& acc, unsigned long long a, unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ unsigned long long bf2x2(uint32_t w) {
  return f2pack(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
// one 16-byte weight chunk (8 bf16) against 8 fp32 activations
__device__ __forceinline__ void dot8_f2(unsigned long long& acc, uint4 w, float4 x0, float4 x1) {
  ffma2(acc, bf2x2(w.x), f2pack(x0.x, x0.y));
  ffma2(acc, bf2x2(w.y), f2pack(x0.z, x0.w));
  ffma2(acc, bf2x2(w.z), f2pack(x1.x, x1.y));
  ffma2(acc, bf2x2(w.w), f2pack(x1.z, x1.w));
}

// gate_up row pair for NT <= 4 tokens with fp32 activations (u32: [B][d]).
template <int NT>
__device__ inline void gu_compute_f32(const uint16_t* gs, const uint16_t* us_rows, const float* u32, uint32_t d,
                                      const Item& it, uint32_t r, float* h_item, uint32_t Fmax) {
  const int lane = lane_id();
  const uint32_t nvec = d / 8;
  unsigned long long ag[NT], au[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) { ag[t] = 0ull; au[t] = 0ull; }
#pragma unroll 2
  for (uint32_t c = lane; c < nvec; c += 32) {
    const uint4 g = reinterpret_cast<const uint4*>(gs)[c];
    const uint4 uu = reinterpret_cast<const uint4*>(us_rows)[c];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      if ((uint32_t)t < it.n_tok) {
        const float4* xp = reinterpret_cast<const float4*>(u32 + (size_t)it.tok[t] * d + c * 8);
        const float4 x0 = xp[0], x1 = xp[1];
        dot8_f2(ag[t], g, x0, x1);
        dot8_f2(au[t], uu, x0, x1);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if ((uint32_t)t < it.n_tok) {
      const float gsum = warp_sum(f2sum(ag[t]));
      const float usum = warp_sum(f2sum(au[t]));
      if (lane == (t & 31)) {
        const float silu = __fdiv_rn(gsum, 1.0f + expf(-gsum));
        h_item[(size_t)t * Fmax + r] = silu * usum;
      }
    }
  }
}

template <int NT>
__device__ inline void gu_compute(const uint16_t* gs, const uint16_t* us_rows, const uint16_t* us, uint32_t d,
                                  const Item& it, uint32_t r, float* h_item, uint32_t Fmax) {
  // gs: gate row in smem; us_rows: up row in smem; us: u [B][d] in smem
  const int lane = lane_id();
  const uint32_t nvec = d / 8;
  float ag[NT], au[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) { ag[t] = 0.f; au[t] = 0.f; }
  for (uint32_t c = lane; c < nvec; c += 32) {
    const uint4 g = reinterpret_cast<const uint4*>(gs)[c];
    const uint4 uu = reinterpret_cast<const uint4*>(us_rows)[c];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      if ((uint32_t)t < it.n_tok) {
        const uint4 xv = reinterpret_cast<const uint4*>(us + (size_t)it.tok[t] * d)[c];
        ag[t] += dot8(g, xv);
        au[t] += dot8(uu, xv);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if ((uint32_t)t < it.n_tok) {
      const float gsum = warp_sum(ag[t]);
      const float usum = warp_sum(au[t]);
      if (lane == (t & 31)) {
        const float silu = __fdiv_rn(gsum, 1.0f + expf(-gsum));
        h_item[(size_t)t * Fmax + r] = silu * usum;
      }
    }
  }
}

template <int NT>
__device__ inline void dn_compute(const uint16_t* ws, const float* hsrc, uint32_t hstride, uint32_t F,
                                  const Item& it, float* acc_row, uint32_t t0 = 0) {
  const int lane = lane_id();
  const uint32_t nvec = F / 8;
  float a[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) a[t] = 0.f;
  // h comes from L2/L1: issue a batch of independent loads before the math
  constexpr int U = NT <= 1 ? 4 : 2;
  if constexpr (NT >= 8) {
    for (uint32_t c = lane; c < nvec; c += 32) {
      const uint4 wv = reinterpret_cast<const uint4*>(ws)[c];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if ((uint32_t)t + t0 < it.n_tok) {
          const float4* hp = reinterpret_cast<const float4*>(hsrc + (size_t)(t + t0) * hstride + c * 8);
          a[t] += dot8f(wv, hp[0], hp[1]);
        }
      }
    }
  } else {
  for (uint32_t c0 = lane; c0 < nvec; c0 += 32 * U) {
    uint4 wv[U];
    float4 h0[U][NT], h1[U][NT];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint32_t c = c0 + 32 * j;
      if (c < nvec) {
        wv[j] = reinterpret_cast<const uint4*>(ws)[c];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if ((uint32_t)t + t0 < it.n_tok) {
            const float4* hp = reinterpret_cast<const float4*>(hsrc + (size_t)(t + t0) * hstride + c * 8);
            h0[j][t] = hp[0];
            h1[j][t] = hp[1];
          }
        }
      }
    }
    unsigned long long a2[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) a2[t] = 0ull;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint32_t c = c0 + 32 * j;
      if (c < nvec) {
#pragma unroll
        for (int t = 0; t < NT; ++t)
          if ((uint32_t)t + t0 < it.n_tok) dot8_f2(a2[t], wv[j], h0[j][t], h1[j][t]);
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) a[t] += f2sum(a2[t]);
  }
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if ((uint32_t)t + t0 < it.n_tok) {
      const float s = warp_sum(a[t]);
      if (lane == 0) {
        const uint32_t tok = it.tok[t + t0];
        acc_row[tok] = fmaf(it.wt[t + t0], s, acc_row[tok]);
      }
    }
  }
}

// gate_up row pair for one token with the fp32 activations held in
// registers (xr: chunk c = lane + 32 j, j < 8, packed f32x2 pairs), which
// covers d <= 2048; wider rows take the remaining chunks from shared memory.
__device__ __forceinline__ unsigned long long bf2x2_asm(uint32_t w) {
  unsigned long long r;
  asm("{\n\t.reg .b32 lo, hi;\n\tshl.b32 lo, %1, 16;\n\tand.b32 hi, %1, 0xffff0000;\n\tmov.b64 %0, {lo, hi};\n\t}"
      : "=l"(r) : "r"(w));
  return r;
}
__device__ inline void gu_pair_x1(const uint16_t* gs, const uint16_t* us_rows, const unsigned long long (&xr)[8][4],
                                  const float* u32, uint32_t d, float* h_out) {
  const int lane = lane_id();
  const uint32_t nvec = d / 8;
  unsigned long long ag0 = 0ull, ag1 = 0ull, au0 = 0ull, au1 = 0ull;
  const uint4* g4 = reinterpret_cast<const uint4*>(gs);
  const uint4* u4 = reinterpret_cast<const uint4*>(us_rows);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t c = lane + 32 * j;
    if (c < nvec) {
      const uint4 g = g4[c], u = u4[c];
      ffma2(ag0, bf2x2_asm(g.x), xr[j][0]);
      ffma2(au0, bf2x2_asm(u.x), xr[j][0]);
      ffma2(ag1, bf2x2_asm(g.y), xr[j][1]);
      ffma2(au1, bf2x2_asm(u.y), xr[j][1]);
      ffma2(ag0, bf2x2_asm(g.z), xr[j][2]);
      ffma2(au0, bf2x2_asm(u.z), xr[j][2]);
      ffma2(ag1, bf2x2_asm(g.w), xr[j][3]);
      ffma2(au1, bf2x2_asm(u.w), xr[j][3]);
    }
  }
  for (uint32_t c = lane + 256; c < nvec; c += 32) {
    const uint4 g = g4[c], u = u4[c];
    const float4* xp = reinterpret_cast<const float4*>(u32 + c * 8);
    const float4 x0 = xp[0], x1 = xp[1];
    dot8_f2(ag0, g, x0, x1);
    dot8_f2(au0, u, x0, x1);
  }
  const float gsum = warp_sum(f2sum(ag0) + f2sum(ag1));
  const float usum = warp_sum(f2sum(au0) + f2sum(au1));
  if (lane == 0) {
    const float silu = __fdiv_rn(gsum, 1.0f + expf(-gsum));
    *h_out = silu * usum;
  }
}

// ---- tensor-core GEMV at batch 1 (mma.sync m16n8k16, bf16 -> fp32).
// A weight row is dotted with the activation through a "diagonal" mapping:
// A rows 0-7 are eight 8-column groups of weight row r0 (columns i*8..i*8+7
// and 64+i*8..64+i*8+7 of a 128-column block), A rows 8-15 the same groups
// of row r1, and B column n holds the activation of group n, so D[i][i] and
// D[8+i][i] are the partial dots of r0 / r1 over group i. ldmatrix reads 128
// contiguous bytes per 8x8 matrix (conflict-free on a row-major stage) and
// one ldmatrix.x4 + one mma cover 512 bytes of weights: the CUDA cores do no
// bf16 unpacking. Products are exact in fp32, accumulation is fp32.
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// this lane's ldmatrix row address inside a 128-column block of rows r0 / r1
__device__ __forceinline__ uint32_t diag_addr(uint32_t r0, uint32_t r1) {
  const int lane = lane_id();
  return ((lane & 8) ? r1 : r0) + ((lane >> 4) & 1) * 128 + (lane & 7) * 16;
}
// sum the diagonal partials: returns (dot r0, dot r1) on every lane
__device__ __forceinline__ float2 diag_reduce(const float (&d)[4]) {
  const int lane = lane_id();
  const int i = lane >> 2;
  const bool mine = (lane & 3) == (i >> 1);
  float v0 = mine ? ((i & 1) ? d[1] : d[0]) : 0.f;
  float v1 = mine ? ((i & 1) ? d[3] : d[2]) : 0.f;
  return make_float2(warp_sum(v0), warp_sum(v1));
}
// B fragments of one token's bf16 activation (d <= 4096) in registers:
// block b -> {x32[b*64 + lane], x32[b*64 + 32 + lane]}
constexpr int kXrBlocks = 32;
__device__ inline void gu_pair_mma(const uint16_t* gs, const uint16_t* us_rows, const uint32_t (&xb)[kXrBlocks][2],
                                   uint32_t d, float* h_out) {
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  float acc2[4] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t base = diag_addr(smem_u32(gs), smem_u32(us_rows));
  const uint32_t nb = d / 128;
#pragma unroll
  for (int b = 0; b < kXrBlocks; b += 2) {
    if ((uint32_t)b < nb) {
      uint32_t a[4];
      ldsm_x4(base + b * 256, a);
      mma16816(acc, a, xb[b][0], xb[b][1]);
    }
    if ((uint32_t)b + 1 < nb) {
      uint32_t a[4];
      ldsm_x4(base + (b + 1) * 256, a);
      mma16816(acc2, a, xb[b + 1][0], xb[b + 1][1]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] += acc2[q];
  const float2 gu = diag_reduce(acc);
  if (lane_id() == 0) {
    const float silu = __fdiv_rn(gu.x, 1.0f + expf(-gu.x));
    *h_out = silu * gu.y;
  }
}
// gate_up row pair for up to NT tokens of an item (tokens [t0, t0+NT)) with
// the bf16 activations in shared memory ([B][d]): the diagonal mapping with
// one ldmatrix per 128-column block shared by the tokens and one mma per
// token (B fragments straight from the token's smem row).
template <int NT>
__device__ inline void gu_pair_mma_tok(const uint16_t* gs, const uint16_t* us_rows, const uint16_t* xs, uint32_t d,
                                       const Item& it, uint32_t t0, uint32_t r, float* h_item, uint32_t Fmax) {
  const int lane = lane_id();
  const uint32_t nt = min((uint32_t)NT, it.n_tok - t0);
  float acc[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[t][q] = 0.f;
  const uint32_t* xw[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t)
    xw[t] = reinterpret_cast<const uint32_t*>(xs + (size_t)it.tok[t0 + ((uint32_t)t < nt ? t : 0)] * d) + lane;
  const uint32_t base = diag_addr(smem_u32(gs), smem_u32(us_rows));
  const uint32_t nb = d / 128;
  for (uint32_t b = 0; b < nb; ++b) {
    uint32_t a[4];
    ldsm_x4(base + b * 256, a);
#pragma unroll
    for (int t = 0; t < NT; ++t)
      if ((uint32_t)t < nt) mma16816(acc[t], a, xw[t][b * 64], xw[t][b * 64 + 32]);
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if ((uint32_t)t < nt) {
      const float2 gu = diag_reduce(acc[t]);
      if (lane == 0) h_item[(size_t)(t0 + t) * Fmax + r] = __fdiv_rn(gu.x, 1.0f + expf(-gu.x)) * gu.y;
    }
  }
}

// down rows r0 / r1 (smem) against h split as bf16 hi + lo (smem words:
// hi32[F/2] then lo32[F/2]); returns the two dots on every lane
__device__ inline float2 dn_pair_mma(const uint16_t* w0, const uint16_t* w1, const uint32_t* hw, uint32_t F) {
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  float acc2[4] = {0.f, 0.f, 0.f, 0.f};
  const int lane = lane_id();
  const uint32_t base = diag_addr(smem_u32(w0), smem_u32(w1));
  const uint32_t nb = F / 128, half = F / 2;
#pragma unroll 2
  for (uint32_t b = 0; b < nb; ++b) {
    uint32_t a[4];
    ldsm_x4(base + b * 256, a);
    const uint32_t* hb = hw + b * 64 + lane;
    mma16816(acc, a, hb[0], hb[32]);
    mma16816(acc2, a, hb[half], hb[half + 32]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] += acc2[q];
  return diag_reduce(acc);
}
__device__ __forceinline__ uint32_t pack_bf16x2(uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); }
// fp32 h -> (hi, lo) bf16 words for the down MMA (h = hi + lo to 2^-16)
__device__ __forceinline__ void split_h4(float4 v, uint32_t& hi01, uint32_t& hi23, uint32_t& lo01, uint32_t& lo23) {
  const uint16_t h0 = f32_to_bf16_rne(v.x), h1 = f32_to_bf16_rne(v.y), h2 = f32_to_bf16_rne(v.z), h3 = f32_to_bf16_rne(v.w);
  hi01 = pack_bf16x2(h0, h1);
  hi23 = pack_bf16x2(h2, h3);
  lo01 = pack_bf16x2(f32_to_bf16_rne(v.x - bf2f(h0)), f32_to_bf16_rne(v.y - bf2f(h1)));
  lo23 = pack_bf16x2(f32_to_bf16_rne(v.z - bf2f(h2)), f32_to_bf16_rne(v.w - bf2f(h3)));
}

// Launch shape of the FFN kernel for a model / batch (host side).
struct FfnLaunch {
  void (*fn)(FfnTArgs);
  int threads;
  uint32_t stages, stage_bytes, hbuf_bytes, acc_rows, plan_smem, x_smem;
  size_t smem;
};

// Persistent grouped SwiGLU FFN. NC consumer warps in NC/kGroupWarps groups;
// ring stage k is consumed by group k % groups (several stages in flight on
// the consumer side), warp w of a group takes gate_up row pair w of a stage
// and the down rows with (row - dlo) % kGroupWarps == w. Each group keeps its
// own down accumulators, summed in group order at the end (deterministic).
constexpr int kGroupWarps = 4;
constexpr size_t kFfnSmemMax = 225 * 1024;

template <int NTMAX, int NC>
__global__ void __launch_bounds__(32 * (NC + 1), 1) ffn_tma_kernel(FfnTArgs a) {
  constexpr int NG = NC / kGroupWarps;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages], empty_bar[kMaxStages];
  // dynamic gate_up stages: {item << 16 | rows, first row}; rows == 0 marks
  // the end of a dynamic phase (second word = next ring step)
  __shared__ uint32_t s_stage_hdr[kMaxStages][2];
  __shared__ uint32_t h_off[kMaxItems + 1];   // h staging offsets of the current phase's ready items
  __shared__ uint32_t s_cpre[kMaxItems + 1];  // gate_up chunk prefix of the current phase's ready items
  __shared__ uint32_t s_arrive[kMaxItems + 2];
  __shared__ uint32_t s_hstage, s_phase_sync;
  // PDL: the next layer's gate+decide kernel may be scheduled once every CTA
  // of this grid is running (it waits for our completion before reading)
  asm volatile("griddepcontrol.launch_dependents;");
  if (a.tl && blockIdx.x == 0 && threadIdx.x == 0) a.tl[7] = globaltimer_ns();
  const uint32_t G = gridDim.x, c = blockIdx.x;
  const uint32_t d = a.d, B = a.B, S = a.stages, SB = a.stage_bytes;
  const int warp = warp_id(), lane = lane_id();
  uint64_t* ts = a.tstamp ? a.tstamp + (size_t)c * 8 : nullptr;
  unsigned char* ring = smem_raw;                                   // S * SB
  uint16_t* us = reinterpret_cast<uint16_t*>(smem_raw + S * SB);  // [B][d] bf16, or [B][d] fp32 when B <= 4
  float* u32 = reinterpret_cast<float*>(us);
  constexpr bool kF32U = false;  // activations stay bf16 in smem (tensor-core gate_up)
  // the plan header + items live in shared memory for the whole launch
  Plan* p = reinterpret_cast<Plan*>(smem_raw + S * SB + a.x_smem);
  float* acc_s = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(p) + a.plan_smem);  // [NG][acc_rows][B]
  const uint32_t acc_n = a.acc_rows * B;
  float* hs = acc_s + ((NG * acc_n + 3) & ~3u);  // h of the current phase's ready items
  const uint32_t gu_rows = min((uint32_t)kGroupWarps, max(1u, SB / (4u * d)));  // row pairs per stage
  uint32_t dlo, dhi;
  share(d, c, G, dlo, dhi);

  // ---- set-up that depends on nothing the decide kernel writes
  for (uint32_t i = threadIdx.x; i < kMaxItems + 2; i += blockDim.x) s_arrive[i] = 0;
  for (uint32_t i = threadIdx.x; i < NG * acc_n; i += blockDim.x) acc_s[i] = 0.f;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kGroupWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // this thread's residual inputs for the epilogue (the previous FFN wrote
  // x_in and has completed: the decide kernel in between waited for it)
  constexpr uint32_t kXinPre = 2;
  float xin_pre[kXinPre];
#pragma unroll
  for (uint32_t j = 0; j < kXinPre; ++j) {
    const uint32_t i = threadIdx.x + j * blockDim.x;
    xin_pre[j] = i < (dhi - dlo) * B ? bf2f(a.x_in[(size_t)(i % B) * d + dlo + i / B]) : 0.f;
  }

  // ---- speculative phase: wait for the decide kernel's early plan
  uint32_t n_spec = 0;
  if (a.spec_plan) {
    if (threadIdx.x == 0) {
      if (ts) ts[0] = globaltimer_ns();
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_u32(a.spec_flag) != a.seq) {
        __nanosleep(64);
        if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 5u); break; }
      }
      if (a.tl && c == 0) a.tl[6] = globaltimer_ns();
    }
    __syncthreads();
    const uint32_t ns = ld_acquire_u32(&a.spec_plan->n_spec);
    const uint64_t* src = reinterpret_cast<const uint64_t*>(a.spec_plan);
    uint64_t* dst = reinterpret_cast<uint64_t*>(p);
    const uint32_t words = (uint32_t)((offsetof(Plan, items) + ns * sizeof(Item)) / 8);
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = __ldcg(src + i);
    n_spec = ns;
  }
  const bool after_spec = a.spec_plan != nullptr;  // the final plan is read after griddepcontrol.wait
  if (!after_spec) {
    // PDL: the plan and u come from the gate+decide kernel launched just before
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (ts && threadIdx.x == 0) ts[0] = globaltimer_ns();
  }
  // u: written by the gate phase before the decider was elected (and
  // released with the spec flag)
  if (!a.x_smem) {
  } else if (kF32U) {
    for (uint32_t i = threadIdx.x; i < B * d / 2; i += blockDim.x) {
      const uint32_t w = __ldcg(reinterpret_cast<const uint32_t*>(a.u) + i);
      u32[2 * i] = __uint_as_float(w << 16);
      u32[2 * i + 1] = __uint_as_float(w & 0xffff0000u);
    }
  } else {
    for (uint32_t i = threadIdx.x; i < B * d / 8; i += blockDim.x)
      reinterpret_cast<uint4*>(us)[i] = __ldcg(reinterpret_cast<const uint4*>(a.u) + i);
  }
  if (!after_spec) {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(a.plan);
    uint64_t* dst = reinterpret_cast<uint64_t*>(p);
    for (uint32_t i = threadIdx.x; i < a.plan_smem / 8; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  if (a.tl && c == 0 && threadIdx.x == 0 && !after_spec) a.tl[0] = globaltimer_ns();

  // Phase bookkeeping (thread 0): gate_up chunks and h staging offsets of
  // the phase's ready items [g0, nr)
  auto setup_phase = [&](uint32_t g0, uint32_t nr) {
    if (threadIdx.x == 0) {
      uint32_t off = 0, ch = 0;
      for (uint32_t i = g0; i < nr; ++i) {
        h_off[i] = off;
        s_cpre[i] = ch;
        off += p->items[i].F * p->items[i].n_tok;
        ch += (p->items[i].F + gu_rows - 1) / gu_rows;
      }
      h_off[nr] = off;
      s_cpre[nr] = ch;
      s_hstage = (size_t)off * 4 <= a.hbuf_bytes;
    }
  };
  auto dn_step = [&](uint32_t F) { return min(4u * kGroupWarps, max(1u, SB / (F * 2))); };

  // A phase: gate_up of the ready items [g0, nr) in grid-dynamic chunks
  // (counter gctr_i), a grid barrier (counter done_i, counting CTAs), the
  // down rows of those items (this CTA's static share), then the items
  // [nr, ni) that wait for their uploads — per item: static gate_up share,
  // grid barrier on ctr[item], down share.
  uint32_t k = 0;  // ring step (producer) / this group's next ring step (consumers)
  const uint32_t cw = warp - 1, grp = cw / kGroupWarps, wg = cw % kGroupWarps;
  if (warp > 0) k = grp;
  // B == 1: the token's bf16 activation as MMA B fragments in registers
  uint32_t xb[kXrBlocks][2];
  auto load_xb = [&]() {
    const uint32_t* u32w = reinterpret_cast<const uint32_t*>(a.u);
#pragma unroll
    for (int b = 0; b < kXrBlocks; ++b) {
      if ((uint32_t)b < d / 128) {
        xb[b][0] = __ldcg(u32w + b * 64 + lane);
        xb[b][1] = __ldcg(u32w + b * 64 + 32 + lane);
      } else {
        xb[b][0] = xb[b][1] = 0u;
      }
    }
  };
  auto gu_rows_of = [&](const unsigned char* src, const Item& it, uint32_t r, uint32_t n, float* h_item) {
    if (wg >= n || (a.dbg & 1)) return;
    const uint32_t nt = it.n_tok;
    const uint16_t* gs = reinterpret_cast<const uint16_t*>(src) + (size_t)wg * d;
    const uint16_t* ur = reinterpret_cast<const uint16_t*>(src + n * d * 2) + (size_t)wg * d;
    if (NTMAX == 1) {
      gu_pair_mma(gs, ur, xb, d, h_item + r + wg);
    } else {
      // tensor cores, tokens in groups of (up to) 4
      (void)u32;
      for (uint32_t t0 = 0; t0 < nt; t0 += 4) {
        if (nt - t0 <= 1) gu_pair_mma_tok<1>(gs, ur, us, d, it, t0, r + wg, h_item, a.Fmax);
        else gu_pair_mma_tok<4>(gs, ur, us, d, it, t0, r + wg, h_item, a.Fmax);
      }
    }
  };
  auto signal = [&](uint32_t si, uint32_t ci) {  // this warp finished its share; last warp of the CTA signals
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      if (atomicAdd(&s_arrive[si], 1u) == NC - 1) {
        __threadfence();
        atomicAdd(&a.ctr[ci], 1u);
      }
    }
  };
  auto grid_wait = [&](uint32_t ci) {  // one poller per CTA, then every consumer warp
    if (cw == 0 && lane == 0) {
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_u32(&a.ctr[ci]) < G) {
        __nanosleep(20);
        if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 2u); break; }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NC * 32) : "memory");
  };
  auto stage_h = [&](uint32_t i0, uint32_t nr) {  // h of items [i0, nr) -> smem (consumers)
    const uint32_t tid = cw * 32 + lane, tot4 = h_off[nr] / 4;
    constexpr uint32_t kU = 8;
    uint32_t i = i0;  // item of v: v only grows for this thread
    for (uint32_t v0 = tid; v0 < tot4; v0 += kU * NC * 32) {
      float4 rv[kU];
      uint32_t ri[kU];
#pragma unroll
      for (uint32_t q = 0; q < kU; ++q) {
        const uint32_t v = v0 + q * NC * 32;
        if (v < tot4) {
          while (h_off[i + 1] / 4 <= v) ++i;
          const uint32_t loc = v - h_off[i] / 4, qq = p->items[i].F / 4;
          const uint32_t t = loc / qq, j = loc % qq;
          rv[q] = __ldcg(reinterpret_cast<const float4*>(a.h + ((size_t)i * kMaxB + t) * a.Fmax) + j);
          ri[q] = i;
        }
      }
#pragma unroll
      for (uint32_t q = 0; q < kU; ++q) {
        const uint32_t v = v0 + q * NC * 32;
        if (v < tot4) {
          const uint32_t ii2 = ri[q], Fi = p->items[ii2].F;
          if (NTMAX == 1 && Fi % 128 == 0) {
            // bf16 hi / lo words for the tensor-core down pass
            const uint32_t loc = v - h_off[ii2] / 4;
            uint32_t* hw = reinterpret_cast<uint32_t*>(hs + h_off[ii2]);
            uint2 hv, lv;
            split_h4(rv[q], hv.x, hv.y, lv.x, lv.y);
            reinterpret_cast<uint2*>(hw)[loc] = hv;
            reinterpret_cast<uint2*>(hw + Fi / 2)[loc] = lv;
          } else {
            reinterpret_cast<float4*>(hs)[v] = rv[q];
          }
        }
      }
    }
  };
  auto dn_rows = [&](const unsigned char* src, const Item& it, uint32_t ii, uint32_t r, uint32_t n, bool staged,
                     float* acc_g) {
    if (a.dbg & 1) return;
    const uint32_t F = it.F, nt = it.n_tok;
    const float* hsrc = staged ? hs + h_off[ii] : a.h + (size_t)ii * kMaxB * a.Fmax;
    const uint32_t hstride = staged ? F : a.Fmax;
    // rows of this step owned by this warp: (row - dlo) % kGroupWarps == wg
    const uint32_t first = (wg + kGroupWarps - (r - dlo) % kGroupWarps) % kGroupWarps;
    if (NTMAX == 1 && F % 128 == 0 && staged) {
      const uint32_t* hw = reinterpret_cast<const uint32_t*>(hsrc);
      const float wt = it.wt[0];
      const uint32_t tok = it.tok[0];
      for (uint32_t q = first; q < n; q += 2 * kGroupWarps) {
        const uint32_t q1 = q + kGroupWarps < n ? q + kGroupWarps : q;
        const uint16_t* w0 = reinterpret_cast<const uint16_t*>(src) + (size_t)q * F;
        const uint16_t* w1 = reinterpret_cast<const uint16_t*>(src) + (size_t)q1 * F;
        const float2 dd = dn_pair_mma(w0, w1, hw, F);
        if (lane == 0) {
          float* a0 = acc_g + (size_t)(r + q - dlo) * B + tok;
          *a0 = fmaf(wt, dd.x, *a0);
          if (q1 != q) {
            float* a1 = acc_g + (size_t)(r + q1 - dlo) * B + tok;
            *a1 = fmaf(wt, dd.y, *a1);
          }
        }
      }
    } else {
      for (uint32_t q = first; q < n; q += kGroupWarps) {
        const uint16_t* ws = reinterpret_cast<const uint16_t*>(src) + (size_t)q * F;
        float* acc_row = acc_g + (size_t)(r + q - dlo) * B;
        // tokens in groups of (up to) 8: no 32-wide accumulator arrays
        for (uint32_t t0 = 0; t0 < nt; t0 += 8) {
          if (NTMAX == 1 || nt - t0 <= 1) dn_compute<1>(ws, hsrc, hstride, F, it, acc_row, t0);
          else if (NTMAX <= 4 || nt - t0 <= 4) dn_compute<(NTMAX < 4 ? NTMAX : 4)>(ws, hsrc, hstride, F, it, acc_row, t0);
          else dn_compute<(NTMAX < 8 ? NTMAX : 8)>(ws, hsrc, hstride, F, it, acc_row, t0);
        }
      }
    }
  };

  auto run_phase = [&](uint32_t g0, uint32_t nr, uint32_t ni, uint32_t gctr_i, uint32_t done_i) {
    if (warp == 0) {
      // --------------------------------------------------------- producer
      if (lane != 0) return;
      const uint64_t pol = l2_evict_first_policy();
      auto acquire = [&]() -> uint32_t {
        const uint32_t st = k % S;
        mbar_wait(&empty_bar[st], ((k / S) & 1) ^ 1);
        return st;
      };
      // (1) gate_up rows of the ready items, chunk by chunk from a grid-wide
      // counter: SMs that stream faster take more chunks (no static skew)
      if (nr > g0) {
        const uint32_t n_chunks = s_cpre[nr];
        uint32_t* gctr = a.ctr + gctr_i;
        uint32_t c0 = atomicAdd(gctr, 1u), c1 = atomicAdd(gctr, 1u);
        uint32_t ii = g0;
        while (c0 < n_chunks) {
          const uint32_t cur = c0;
          c0 = c1;
          c1 = atomicAdd(gctr, 1u);
          while (s_cpre[ii + 1] <= cur) ++ii;
          const Item& it = p->items[ii];
          const uint32_t F = it.F;
          const uint32_t r = (cur - s_cpre[ii]) * gu_rows;
          const uint32_t n = min(gu_rows, F - r);
          const uint32_t st = acquire();
          s_stage_hdr[st][0] = (ii << 16) | n;
          s_stage_hdr[st][1] = r;
          unsigned char* dst = ring + st * SB;
          mbar_expect_tx(&full_bar[st], 2 * n * d * 2);
          bulk_g2s(dst, it.w + (size_t)r * d, n * d * 2, &full_bar[st], pol);
          bulk_g2s(dst + n * d * 2, it.w + ((size_t)F + r) * d, n * d * 2, &full_bar[st], pol);
          ++k;
        }
        const uint32_t k_next = k + NG;
        for (int g = 0; g < NG; ++g) {  // one end marker per consumer group
          const uint32_t st = acquire();
          s_stage_hdr[st][0] = 0;
          s_stage_hdr[st][1] = k_next;
          mbar_arrive(&full_bar[st]);
          ++k;
        }
        // (2) down rows of the ready items (static share)
        for (uint32_t ii2 = g0; ii2 < nr; ++ii2) {
          if (a.dbg & 2) break;
          const Item& it = p->items[ii2];
          const uint32_t F = it.F, step = dn_step(F);
          for (uint32_t r = dlo; r < dhi; r += step) {
            const uint32_t n = min(step, dhi - r);
            const uint32_t st = acquire();
            mbar_expect_tx(&full_bar[st], n * F * 2);
            bulk_g2s(ring + st * SB, it.w + 2 * (size_t)F * d + (size_t)r * F, n * F * 2, &full_bar[st], pol);
            ++k;
          }
        }
      }
      // (3) the waiting items, one at a time
      for (uint32_t ii2 = nr; ii2 < ni; ++ii2) {
        const Item& it = p->items[ii2];
        const uint32_t F = it.F;
        if (it.wait) {
          const uint64_t t0 = globaltimer_ns();
          while ((int32_t)(ld_acquire_u32(a.copies_done) - it.wait) < 0) {
            __nanosleep(128);
            if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 1u); break; }
          }
          if (a.tl && c == 0) a.tl[1] = globaltimer_ns();
          // the uploaded bytes are read by the async (bulk-copy) proxy next
          asm volatile("fence.proxy.async;" ::: "memory");
        }
        uint32_t lo, hi;
        share(F, c, G, lo, hi);
        for (uint32_t r = lo; r < hi; r += gu_rows) {
          const uint32_t n = min(gu_rows, hi - r);
          const uint32_t st = acquire();
          unsigned char* dst = ring + st * SB;
          mbar_expect_tx(&full_bar[st], 2 * n * d * 2);
          bulk_g2s(dst, it.w + (size_t)r * d, n * d * 2, &full_bar[st], pol);
          bulk_g2s(dst + n * d * 2, it.w + ((size_t)F + r) * d, n * d * 2, &full_bar[st], pol);
          ++k;
        }
        if (a.dbg & 2) continue;
        const uint32_t step = dn_step(F);
        for (uint32_t r = dlo; r < dhi; r += step) {
          const uint32_t n = min(step, dhi - r);
          const uint32_t st = acquire();
          mbar_expect_tx(&full_bar[st], n * F * 2);
          bulk_g2s(ring + st * SB, it.w + 2 * (size_t)F * d + (size_t)r * F, n * F * 2, &full_bar[st], pol);
          ++k;
        }
      }
      return;
    }
    // ----------------------------------------------------------- consumers
    // Ring step k (stage k % S) belongs to consumer group k % NG (S is a
    // multiple of NG, so a stage always has the same group and its phases are
    // consumed in order).
    float* acc_g = acc_s + grp * acc_n;
    if (nr > g0) {
      if (NTMAX == 1) load_xb();
      for (;;) {  // (1) dynamic gate_up
        const uint32_t st = k % S;
        mbar_wait(&full_bar[st], (k / S) & 1);
        const uint32_t h0 = s_stage_hdr[st][0], r = s_stage_hdr[st][1];
        const uint32_t n = h0 & 0xffffu;
        if (n == 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[st]);
          k = r + grp;  // r = first step after the end markers; this group's first step
          break;
        }
        const uint32_t ii = h0 >> 16;
        gu_rows_of(ring + st * SB, p->items[ii], r, n, a.h + (size_t)ii * kMaxB * a.Fmax);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
        k += NG;
      }
    }
    if (nr > g0) {
      const bool spec_phase = done_i == kFfnSpecDoneCtr;
      signal(kMaxItems + (spec_phase ? 1 : 0), done_i);
      if (a.tl && c == 0 && cw == 0 && lane == 0) a.tl[spec_phase ? 8 : 9] = globaltimer_ns();
      if (ts && cw == 0 && lane == 0) ts[3] = globaltimer_ns();
      // (2) down rows of the ready items, after every CTA's gate_up
      grid_wait(done_i);
      if (s_hstage) {
        stage_h(g0, nr);
        asm volatile("bar.sync 1, %0;" ::"n"(NC * 32) : "memory");
      }
      if (ts && cw == 0 && lane == 0) ts[4] = globaltimer_ns();
      if (a.tl && c == 0 && cw == 0 && lane == 0 && !spec_phase) a.tl[10] = globaltimer_ns();
      if (!(a.dbg & 2)) {
        // steps are numbered globally: walk them, take this group's
        uint32_t kk = k - grp;  // global step of the first down stage
        for (uint32_t ii = g0; ii < nr; ++ii) {
          const Item& it = p->items[ii];
          const uint32_t F = it.F, step = dn_step(F);
          for (uint32_t r = dlo; r < dhi; r += step, ++kk) {
            const uint32_t st = kk % S;
            if (st % NG != grp) continue;
            mbar_wait(&full_bar[st], (kk / S) & 1);
            dn_rows(ring + st * SB, it, ii, r, min(step, dhi - r), s_hstage != 0, acc_g);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[st]);
          }
        }
        k = kk + grp;
      }
    }
    // (3) the waiting items
    uint32_t kk = k - grp;
    for (uint32_t ii = nr; ii < ni; ++ii) {
      const Item& it = p->items[ii];
      const uint32_t F = it.F;
      float* h_item = a.h + (size_t)ii * kMaxB * a.Fmax;
      uint32_t lo, hi;
      share(F, c, G, lo, hi);
      if (NTMAX == 1) load_xb();
      for (uint32_t r = lo; r < hi; r += gu_rows, ++kk) {
        const uint32_t st = kk % S;
        if (st % NG != grp) continue;
        mbar_wait(&full_bar[st], (kk / S) & 1);
        gu_rows_of(ring + st * SB, it, r, min(gu_rows, hi - r), h_item);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
      }
      signal(ii, ii);
      if (a.dbg & 2) continue;
      grid_wait(ii);
      const uint32_t step = dn_step(F);
      for (uint32_t r = dlo; r < dhi; r += step, ++kk) {
        const uint32_t st = kk % S;
        if (st % NG != grp) continue;
        mbar_wait(&full_bar[st], (kk / S) & 1);
        dn_rows(ring + st * SB, it, ii, r, min(step, dhi - r), false, acc_g);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
      }
    }
    k = kk + grp;
  };

  // ---- the speculative items (gate_up, grid barrier, down rows),
  // overlapped with the rest of the decision
  if (after_spec && n_spec) {
    setup_phase(0, n_spec);
    __syncthreads();
    run_phase(0, n_spec, n_spec, kFfnSpecGuCtr, kFfnSpecDoneCtr);
  }
  if (after_spec) {
    // ---- the final plan: every item after the speculative ones. Taken from
    // the decide kernel's release of spec_flag[1], not griddepcontrol.wait
    // (kernel completion flushes behind this kernel's own weight stream)
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_u32(a.spec_flag + 1) != a.seq) {
        __nanosleep(32);
        if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 6u); break; }
      }
      if (a.tl && c == 0) a.tl[0] = globaltimer_ns();
    }
    __syncthreads();
    const Plan* gp = a.plan;
    if (threadIdx.x < 4) reinterpret_cast<uint32_t*>(p)[threadIdx.x] = __ldcg(reinterpret_cast<const uint32_t*>(gp) + threadIdx.x);
    {
      const uint64_t* src = reinterpret_cast<const uint64_t*>(gp->items + n_spec);
      uint64_t* dst = reinterpret_cast<uint64_t*>(p->items + n_spec);
      const uint32_t words = (uint32_t)((a.plan_smem - offsetof(Plan, items)) / 8 - n_spec * (sizeof(Item) / 8));
      for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = __ldcg(src + i);
    }
    if (threadIdx.x == 0) p->d2d_elems = __ldcg(&gp->d2d_elems);
  }
  // every warp has left the speculative phase and sees the final plan; the
  // down accumulators of the speculative items stay in acc_s
  __syncthreads();
  {
    const uint32_t n_items = p->n_items, n_ready = p->n_ready;
    setup_phase(n_spec, n_ready);
    __syncthreads();
    run_phase(n_spec, n_ready, n_items, kFfnGuCtr, kFfnReadyDoneCtr);
  }
  __syncthreads();
  if (ts && threadIdx.x == 0) ts[5] = globaltimer_ns();
  if (a.tl && c == 0 && threadIdx.x == 0) a.tl[11] = globaltimer_ns();
  // epilogue: group partial sums (fixed order), residual add (x_in was read
  // at the start), bf16 hidden for the next layer, fp32 MoE output
  for (uint32_t i = threadIdx.x, j = 0; i < (dhi - dlo) * B; i += blockDim.x, ++j) {
    const uint32_t o = dlo + i / B, t = i % B;
    float y = acc_s[i];
#pragma unroll
    for (int g = 1; g < NG; ++g) y += acc_s[g * acc_n + i];
    const float xo = (j < kXinPre ? xin_pre[j] : bf2f(a.x_in[(size_t)t * d + o])) + y;
    a.x_out[(size_t)t * d + o] = f32_to_bf16_rne(xo);
    a.y_out[(size_t)t * d + o] = y;
  }
  // deferred admissions: staging -> slot once every CTA finished reading
  const uint32_t n_d2d = p->n_d2d;
  if (n_d2d) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&a.ctr[kFfnD2dCtr], 1u);
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_u32(&a.ctr[kFfnD2dCtr]) < G) {
        __nanosleep(128);
        if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 3u); break; }
      }
    }
    __syncthreads();
    const Plan* gp = a.plan;
    const uint64_t nv = p->d2d_elems / 8;
    for (uint32_t j = 0; j < n_d2d; ++j) {
      const uint4* src = reinterpret_cast<const uint4*>(__ldcg(reinterpret_cast<const unsigned long long*>(&gp->d2d[j].src)));
      uint4* dst = reinterpret_cast<uint4*>(__ldcg(reinterpret_cast<const unsigned long long*>(&gp->d2d[j].dst)));
      for (uint64_t v = c * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)G * blockDim.x)
        dst[v] = ldg_cg(src + v);
    }
  }
  __syncthreads();
  if (ts && threadIdx.x == 0) ts[7] = globaltimer_ns();
  if (threadIdx.x == 0) {
    // slot reads are complete (they landed in smem); only the deferred
    // staging->slot copies must be visible before ffn_done releases the
    // copy stream's prefetches into those slots
    if (n_d2d) __threadfence();
    const uint32_t prev = atomicAdd(&a.ctr[kFfnExitCtr], 1u);
    if (prev == G - 1) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ffn_done), "r"(p->seq) : "memory");
      if (a.tl) a.tl[2] = globaltimer_ns();
    }
    if (ts) ts[6] = globaltimer_ns();
  }
}

// Kernel instance and shared-memory layout for a model / batch. Throws
// nothing: returns stages == 0 when the shapes do not fit.
inline FfnLaunch ffn_launch_config(uint32_t B, uint32_t d, uint32_t F, uint32_t S, uint32_t E, uint32_t top_k,
                                   int grid) {
  const int sms = grid;  // CTAs of the persistent grid
  FfnLaunch L{};
  int nc;
  if (B <= 1) { L.fn = ffn_tma_kernel<1, 12>; nc = 12; }
  else if (B <= 4) { L.fn = ffn_tma_kernel<4, 12>; nc = 12; }
  else if (B <= 8) { L.fn = ffn_tma_kernel<8, 8>; nc = 8; }
  else if (B <= 16) { L.fn = ffn_tma_kernel<16, 8>; nc = 8; }
  else { L.fn = ffn_tma_kernel<32, 8>; nc = 8; }
  L.threads = 32 * (nc + 1);
  const uint32_t ng = nc / kGroupWarps;
  const uint32_t max_items = 1 + std::min(E, B * top_k);
  L.plan_smem = (uint32_t)((offsetof(Plan, items) + (size_t)max_items * sizeof(Item) + 15) & ~(size_t)15);
  L.x_smem = (B == 1 && d <= 2048) ? 0u : (uint32_t)((((size_t)B * d * 2) + 15) & ~(size_t)15);
  L.acc_rows = (d + sms - 1) / sms;
  const size_t accb = ((size_t)ng * L.acc_rows * B + 3) / 4 * 16;
  const size_t fixed = L.x_smem + L.plan_smem + accb;
  const size_t pair = 4ull * d;  // one gate + one up row
  // h of the ready items (shared + top-k experts x tokens) staged in smem
  // when it fits beside one ring stage of one pair per group
  const size_t hwant = ((size_t)S + (size_t)top_k * F) * B * 4;
  const size_t min_ring = 2ull * ng * std::max<size_t>(pair, (2 * std::max(F, S) + 1023) / 1024 * 1024);
  L.hbuf_bytes = (uint32_t)(kFfnSmemMax >= fixed + min_ring + hwant ? hwant : 0);
  const size_t budget = kFfnSmemMax - fixed - L.hbuf_bytes;
  // two stages per consumer group; a stage holds up to kGroupWarps gate+up
  // row pairs and at least one down row (2 * ffn bytes) and one pair
  const size_t fmax = std::max(F, S);
  const size_t min_sb = std::max<size_t>(pair, (2 * fmax + 1023) / 1024 * 1024);
  size_t sb = budget / (2 * ng) / pair * pair;
  if (sb > kGroupWarps * pair) sb = kGroupWarps * pair;
  if (sb < min_sb) sb = min_sb;
  uint32_t st = (uint32_t)std::min<size_t>(kMaxStages, budget / sb);
  st -= st % ng;  // a stage always belongs to the same consumer group
  L.stage_bytes = (uint32_t)sb;
  L.stages = st >= ng ? st : 0;
  L.smem = (size_t)L.stages * L.stage_bytes + fixed + L.hbuf_bytes;
  return L;
}

}  // namespace moeb
