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

#include <cstdint>
#include <cuda_runtime.h>

#include "layer.cuh"

namespace moeb {

constexpr int kConsumers = 8;
constexpr int kFfnTThreads = 32 * (1 + kConsumers);
constexpr int kMaxStages = 8;
constexpr uint32_t kHbufBytes = 48 * 1024;   // h staged in smem when it fits
constexpr int kMaxDnRowsPerCta = 64;
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
  float* h;                // [kMaxItems][B][Fmax]
  uint32_t* ctr;           // [0,kMaxItems) item gate_up done, [kMaxItems] d2d barrier, [kMaxItems+1] exit
  const uint32_t* copies_done;
  uint32_t* ffn_done;
  uint32_t B, d, Fmax, stages;
  uint32_t stage_bytes;    // bytes per ring stage (multiple of 1 KB)
  uint32_t hbuf_bytes;     // smem reserved for staging h of the ready items
  uint32_t dbg;            // microbenchmark knobs: 1 no consumer math, 2 skip down pass
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
                                  const Item& it, float* acc_row) {
  const int lane = lane_id();
  const uint32_t nvec = F / 8;
  float a[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) a[t] = 0.f;
  // h comes from L2/L1: issue a batch of independent loads before the math
  constexpr int U = NT <= 1 ? 6 : 2;
  if constexpr (NT >= 8) {
    for (uint32_t c = lane; c < nvec; c += 32) {
      const uint4 wv = reinterpret_cast<const uint4*>(ws)[c];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if ((uint32_t)t < it.n_tok) {
          const float4* hp = reinterpret_cast<const float4*>(hsrc + (size_t)t * hstride + c * 8);
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
          if ((uint32_t)t < it.n_tok) {
            const float4* hp = reinterpret_cast<const float4*>(hsrc + (size_t)t * hstride + c * 8);
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
          if ((uint32_t)t < it.n_tok) dot8_f2(a2[t], wv[j], h0[j][t], h1[j][t]);
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) a[t] += f2sum(a2[t]);
  }
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if ((uint32_t)t < it.n_tok) {
      const float s = warp_sum(a[t]);
      if (lane == 0) {
        const uint32_t tok = it.tok[t];
        acc_row[tok] = fmaf(it.wt[t], s, acc_row[tok]);
      }
    }
  }
}

template <int NTMAX>
__global__ void __launch_bounds__(kFfnTThreads, 1) ffn_tma_kernel(FfnTArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages], empty_bar[kMaxStages];
  __shared__ float acc_s[kMaxDnRowsPerCta * kMaxB];
  __shared__ uint32_t s_hdr[4];
  // PDL: the plan and u come from the gate+decide kernel launched just before
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const Plan* gp = a.plan;
  const uint32_t G = gridDim.x, c = blockIdx.x;
  const uint32_t d = a.d, B = a.B, S = a.stages, SB = a.stage_bytes;
  const int warp = warp_id(), lane = lane_id();
  unsigned char* ring = smem_raw;                                   // S * 32 KB
  uint16_t* us = reinterpret_cast<uint16_t*>(smem_raw + S * SB);  // [B][d] bf16, or [B][d] fp32 when B <= 4
  float* u32 = reinterpret_cast<float*>(us);
  constexpr bool kF32U = NTMAX <= 4;
  // the plan header + items live in shared memory for the whole launch
  Plan* p = reinterpret_cast<Plan*>(smem_raw + S * SB + (((size_t)B * d * (kF32U ? 4 : 2) + 15) & ~(size_t)15));
  if (threadIdx.x < 4) s_hdr[threadIdx.x] = reinterpret_cast<const uint32_t*>(gp)[threadIdx.x];
  __syncthreads();
  {
    const size_t words = (offsetof(Plan, items) + s_hdr[0] * sizeof(Item)) / 8;
    const uint64_t* src = reinterpret_cast<const uint64_t*>(gp);
    uint64_t* dst = reinterpret_cast<uint64_t*>(p);
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
    const size_t d0 = offsetof(Plan, d2d) / 8, d1 = d0 + s_hdr[2] * sizeof(D2D) / 8;
    for (uint32_t i = d0 + threadIdx.x; i < d1; i += blockDim.x) dst[i] = src[i];
  }
  const uint32_t n_items = s_hdr[0], n_ready = s_hdr[1];
  // h of every ready item, staged once after the ready gate_up barrier
  float* hs = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(p) + kPlanSmem);
  __shared__ uint32_t h_off[kMaxItems + 1];
  __shared__ uint32_t s_hstage;
  const uint32_t gu_rows = min((uint32_t)kConsumers, max(1u, SB / (4u * d)));  // row pairs per stage

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (kF32U) {
    for (uint32_t i = threadIdx.x; i < B * d / 2; i += blockDim.x) {
      const uint32_t w = reinterpret_cast<const uint32_t*>(a.u)[i];
      u32[2 * i] = __uint_as_float(w << 16);
      u32[2 * i + 1] = __uint_as_float(w & 0xffff0000u);
    }
  } else {
    for (uint32_t i = threadIdx.x; i < B * d / 8; i += blockDim.x)
      reinterpret_cast<uint4*>(us)[i] = reinterpret_cast<const uint4*>(a.u)[i];
  }
  uint32_t dlo, dhi;
  share(d, c, G, dlo, dhi);
  for (uint32_t i = threadIdx.x; i < (dhi - dlo) * B; i += blockDim.x) acc_s[i] = 0.f;
  if (threadIdx.x == 0) {
    uint32_t off = 0;
    for (uint32_t i = 0; i < n_ready; ++i) {
      h_off[i] = off;
      off += p->items[i].F * p->items[i].n_tok;
    }
    h_off[n_ready] = off;
    s_hstage = (size_t)off * 4 <= a.hbuf_bytes;
  }
  __syncthreads();

  // enumerate (item, kind) segments in schedule order
  auto seg_item = [&](uint32_t s, uint32_t& item, uint32_t& kind) {
    if (s < n_ready) { item = s; kind = 0; return; }
    s -= n_ready;
    if (s < n_ready) { item = s; kind = 1; return; }
    s -= n_ready;
    item = n_ready + s / 2;
    kind = s & 1;
  };
  const uint32_t n_segs = 2 * n_items;
  auto skip_seg = [&](uint32_t sg) {
    uint32_t ii, kind;
    seg_item(sg, ii, kind);
    return (a.dbg & 2) && kind == 1;
  };

  if (warp == 0) {
    // ------------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      uint32_t stage = 0, phase = 0;
      for (uint32_t sg = 0; sg < n_segs; ++sg) {
        if (skip_seg(sg)) continue;
        uint32_t ii, kind;
        seg_item(sg, ii, kind);
        const Item& it = p->items[ii];
        const uint32_t F = it.F;
        if (kind == 0 && it.wait) {
          const uint64_t t0 = globaltimer_ns();
          while ((int32_t)(ld_acquire_u32(a.copies_done) - it.wait) < 0) {
            __nanosleep(128);
            if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 1u); break; }
          }
          // the uploaded bytes are read by the async (bulk-copy) proxy next
          asm volatile("fence.proxy.async;" ::: "memory");
        }
        uint32_t lo, hi, step, row_bytes;
        if (kind == 0) {
          share(F, c, G, lo, hi);
          step = gu_rows;
          row_bytes = d * 2;
        } else {
          lo = dlo;
          hi = dhi;
          step = min((uint32_t)kConsumers, max(1u, SB / (F * 2)));
          row_bytes = F * 2;
        }
        for (uint32_t r = lo; r < hi; r += step) {
          const uint32_t n = min(step, hi - r);
          mbar_wait(&empty_bar[stage], phase ^ 1);
          unsigned char* dst = ring + stage * SB;
          if (kind == 0) {
            const uint16_t* g = it.w + (size_t)r * d;
            const uint16_t* u = it.w + ((size_t)F + r) * d;
            mbar_expect_tx(&full_bar[stage], 2 * n * row_bytes);
            bulk_g2s(dst, g, n * row_bytes, &full_bar[stage], pol);
            bulk_g2s(dst + n * row_bytes, u, n * row_bytes, &full_bar[stage], pol);
          } else {
            const uint16_t* w = it.w + 2 * (size_t)F * d + (size_t)r * F;
            mbar_expect_tx(&full_bar[stage], n * row_bytes);
            bulk_g2s(dst, w, n * row_bytes, &full_bar[stage], pol);
          }
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ------------------------------------------------------ consumers
    // Each consumer warp signals its own completion of an item's gate_up rows
    // (ctr[i] counts warps, G * kConsumers when complete) and waits on its
    // own for the down pass: no CTA-wide barriers between items. h is read
    // straight from global after the acquire (it is tiny and L1-resident).
    const uint32_t cw = warp - 1;
    uint32_t stage = 0, phase = 0;
    for (uint32_t sg = 0; sg < n_segs; ++sg) {
      if (skip_seg(sg)) continue;
      uint32_t ii, kind;
      seg_item(sg, ii, kind);
      const Item& it = p->items[ii];
      const uint32_t F = it.F, nt = it.n_tok;
      float* h_item = a.h + (size_t)ii * kMaxB * a.Fmax;
      uint32_t lo, hi, step;
      const float* hsrc = h_item;
      uint32_t hstride = a.Fmax;
      if (kind == 0) {
        share(F, c, G, lo, hi);
        step = gu_rows;
      } else {
        lo = dlo;
        hi = dhi;
        step = min((uint32_t)kConsumers, max(1u, SB / (F * 2)));
        // ready items signal once, on ctr[0] after the last ready gate_up
        // segment; each waiting item has its own counter
        const bool ready = ii < n_ready;
        const bool first_dn = ready && sg == n_ready;  // first down segment of the ready group
        if (!ready || first_dn) {
          const uint32_t wc = ready ? 0 : ii;
          if (lane == 0) {
            const uint64_t t0 = globaltimer_ns();
            while (ld_acquire_u32(&a.ctr[wc]) < G * kConsumers) {
              __nanosleep(32);
              if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 2u); break; }
            }
          }
          __syncwarp();
        }
        if (first_dn && s_hstage) {
          // stage h of all ready items into shared memory in one batch
          asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
          const uint32_t tid = cw * 32 + lane;
          for (uint32_t i = 0; i < n_ready; ++i) {
            const Item& ri = p->items[i];
            const uint32_t q = ri.F / 4;
            const float* hb = a.h + (size_t)i * kMaxB * a.Fmax;
            for (uint32_t v = tid; v < ri.n_tok * q; v += kConsumers * 32) {
              const uint32_t t = v / q, j = v % q;
              reinterpret_cast<float4*>(hs + h_off[i])[v] =
                  __ldcg(reinterpret_cast<const float4*>(hb + (size_t)t * a.Fmax) + j);
            }
          }
          asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
        }
        if (ready && s_hstage) {
          hsrc = hs + h_off[ii];
          hstride = F;
        }
      }
      for (uint32_t r = lo; r < hi; r += step) {
        const uint32_t n = min(step, hi - r);
        mbar_wait(&full_bar[stage], phase);
        const unsigned char* src = ring + stage * SB;
        if (cw < n && !(a.dbg & 1)) {
          if (kind == 0) {
            const uint16_t* gs = reinterpret_cast<const uint16_t*>(src) + (size_t)cw * d;
            const uint16_t* ur = reinterpret_cast<const uint16_t*>(src + n * d * 2) + (size_t)cw * d;
            if (kF32U) {
              if (NTMAX == 1 || nt <= 1) gu_compute_f32<1>(gs, ur, u32, d, it, r + cw, h_item, a.Fmax);
              else gu_compute_f32<(NTMAX < 4 ? NTMAX : 4)>(gs, ur, u32, d, it, r + cw, h_item, a.Fmax);
            }
            else if (NTMAX <= 4 || nt <= 4) gu_compute<(NTMAX < 4 ? NTMAX : 4)>(gs, ur, us, d, it, r + cw, h_item, a.Fmax);
            else if (NTMAX <= 8 || nt <= 8) gu_compute<(NTMAX < 8 ? NTMAX : 8)>(gs, ur, us, d, it, r + cw, h_item, a.Fmax);
            else gu_compute<NTMAX>(gs, ur, us, d, it, r + cw, h_item, a.Fmax);
          } else {
            const uint16_t* ws = reinterpret_cast<const uint16_t*>(src) + (size_t)cw * F;
            float* acc_row = acc_s + (size_t)(r + cw - dlo) * B;
            if (NTMAX == 1 || nt <= 1) dn_compute<1>(ws, hsrc, hstride, F, it, acc_row);
            else if (NTMAX <= 4 || nt <= 4) dn_compute<(NTMAX < 4 ? NTMAX : 4)>(ws, hsrc, hstride, F, it, acc_row);
            else if (NTMAX <= 8 || nt <= 8) dn_compute<(NTMAX < 8 ? NTMAX : 8)>(ws, hsrc, hstride, F, it, acc_row);
            else dn_compute<NTMAX>(ws, hsrc, hstride, F, it, acc_row);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[stage]);
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
      if (kind == 0 && (ii >= n_ready || ii + 1 == n_ready)) {
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          atomicAdd(&a.ctr[ii < n_ready ? 0 : ii], 1u);
        }
      }
    }
  }
  __syncthreads();
  // epilogue: residual add, bf16 hidden for the next layer, fp32 MoE output
  for (uint32_t i = threadIdx.x; i < (dhi - dlo) * B; i += blockDim.x) {
    const uint32_t o = dlo + i / B, t = i % B;
    const float y = acc_s[i];
    const float xo = bf2f(a.x_in[(size_t)t * d + o]) + y;
    a.x_out[(size_t)t * d + o] = f32_to_bf16_rne(xo);
    a.y_out[(size_t)t * d + o] = y;
  }
  // deferred admissions: staging -> slot once every CTA finished reading
  if (p->n_d2d) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&a.ctr[kMaxItems], 1u);
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_u32(&a.ctr[kMaxItems]) < G) {
        __nanosleep(128);
        if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 3u); break; }
      }
    }
    __syncthreads();
    const uint64_t nv = p->d2d_elems / 8;
    for (uint32_t j = 0; j < p->n_d2d; ++j) {
      const uint4* src = reinterpret_cast<const uint4*>(p->d2d[j].src);
      uint4* dst = reinterpret_cast<uint4*>(p->d2d[j].dst);
      for (uint64_t v = c * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)G * blockDim.x)
        dst[v] = ldg_cg(src + v);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(&a.ctr[kMaxItems + 1], 1u);
    if (prev == G - 1) {
      __threadfence_system();
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.ffn_done), "r"(p->seq) : "memory");
    }
  }
}

}  // namespace moeb
