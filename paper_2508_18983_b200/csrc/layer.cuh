// layer.cuh — the MoE layer arithmetic kernels (sm_100a).
//
//   gate_kernel : RMSNorm (fp32) -> u (bf16) and router GEMV logits = Wg.u
//                 (fp32 accumulate over bf16 weights), plus the Qwen shared-
//                 expert gate row. HBM-bound: E*d*2 bytes per layer.
//   ffn_kernel  : persistent grouped SwiGLU over the plan's items (shared
//                 expert + every distinct selected expert, each with its token
//                 list and combine weights): gate_up GEMV -> silu(g)*u -> down
//                 GEMV -> weighted, deterministic combine + residual. Items
//                 whose weights are still on the PCIe copy stream are waited
//                 for item by item, so resident-expert work overlaps uploads.
//                 HBM-bound at decode (AI <= ~3 FLOP/B for B <= 32).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "engine.cuh"
#include "weights.cuh"

namespace moeb {

constexpr int kMaxItems = 1 + kMaxE;
constexpr int kFfnWarps = 16;
constexpr int kFfnThreads = kFfnWarps * 32;
constexpr int kGateThreads = 256;

struct Item {
  const uint16_t* w;  // [gate F*d][up F*d][down d*F] bf16
  uint32_t F;
  uint32_t wait;      // upload id the weights depend on (0 = ready)
  uint32_t n_tok;
  uint32_t kind;      // 0 shared, 1 resident, 2 loaded, 3 streamed
  uint32_t expert;
  uint32_t spec;      // (buffer << 31) | generation: weights come from a speculative upload
                      // buffer, ready once spec_done[buffer] >= generation (0: none)
  uint8_t tok[kMaxB];
  float wt[kMaxB];
};
struct D2D {
  const uint16_t* src;
  uint16_t* dst;
};
struct Plan {
  uint32_t n_items, n_ready, n_d2d, seq;
  uint64_t d2d_elems;
  uint32_t n_spec;    // items [0, n_spec) were published early (speculative plan)
  uint32_t n_local;   // items [0, n_local) are the shared expert + resident hits (kind <= 1)
  Item items[kMaxItems];
  D2D d2d[kMaxE];
};

// --------------------------------------------------------------- helpers
__device__ __forceinline__ float bf2f(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }
__device__ __forceinline__ uint4 ldg_cg(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float dot8(uint4 w, uint4 x) {
  const uint32_t a[4] = {w.x, w.y, w.z, w.w};
  const uint32_t b[4] = {x.x, x.y, x.z, x.w};
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s = fmaf(__uint_as_float(a[i] << 16), __uint_as_float(b[i] << 16), s);
    s = fmaf(__uint_as_float(a[i] & 0xffff0000u), __uint_as_float(b[i] & 0xffff0000u), s);
  }
  return s;
}
__device__ __forceinline__ float dot8f(uint4 w, float4 h0, float4 h1) {
  float s = 0.f;
  s = fmaf(__uint_as_float(w.x << 16), h0.x, s);
  s = fmaf(__uint_as_float(w.x & 0xffff0000u), h0.y, s);
  s = fmaf(__uint_as_float(w.y << 16), h0.z, s);
  s = fmaf(__uint_as_float(w.y & 0xffff0000u), h0.w, s);
  s = fmaf(__uint_as_float(w.z << 16), h1.x, s);
  s = fmaf(__uint_as_float(w.z & 0xffff0000u), h1.y, s);
  s = fmaf(__uint_as_float(w.w << 16), h1.z, s);
  s = fmaf(__uint_as_float(w.w & 0xffff0000u), h1.w, s);
  return s;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Spins are bounded: a lost upload must not hang the GPU. After kSpinLimitNs
// the waiter gives up and raises the sticky error flag the host checks.
constexpr uint64_t kSpinLimitNs = 20ull * 1000 * 1000 * 1000;
__device__ uint32_t g_spin_timeout;

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Deterministic softmax of one token's logits by one warp (lanes hold
// experts lane, lane+32). Butterfly sums are symmetric, so every lane holds
// the bit-identical total; division is IEEE round-to-nearest.
__device__ inline void softmax_warp(const float* logits, uint32_t E, float* out) {
  const int lane = lane_id();
  const float l0 = (uint32_t)lane < E ? logits[lane] : -INFINITY;
  const float l1 = (uint32_t)lane + 32 < E ? logits[lane + 32] : -INFINITY;
  float m = fmaxf(l0, l1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float x0 = (uint32_t)lane < E ? expf(l0 - m) : 0.f;
  const float x1 = (uint32_t)lane + 32 < E ? expf(l1 - m) : 0.f;
  float s = x0 + x1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((uint32_t)lane < E) out[lane] = __fdiv_rn(x0, s);
  if ((uint32_t)lane + 32 < E) out[lane + 32] = __fdiv_rn(x1, s);
}

// ------------------------------------------------------------------ gate
struct GateArgs {
  const uint16_t* x;       // [B][d] bf16 layer input
  const uint16_t* wg;      // [E][d] router weights of this layer
  const uint16_t* wsg;     // [d] Qwen shared-expert gate row (nullable)
  uint16_t* u;             // [B][d] normalised input (written by CTA 0)
  uint16_t* ut;            // the same, SW128-tiled [d/64][ut_rows][64] for the batched
                           // tensor-core FFN (nullable; written by CTA 1, rows >= B stay 0)
  uint32_t ut_rows;
  float* logits;           // [B][E + 1]; column E = shared-gate logit
  const uint16_t* x_pred;  // [B][d] the previous layer's partial forward (predictor) or null
  float* plogits;          // [B][E + 1]: the same router applied to it
  uint32_t B, d, E;
};

// ng = ceil(rows / 2) gate CTAs with rows = E (+1 for the shared gate), gi the
// CTA's index among them; 8 warps: warp w -> row 2*gi + (w & 1), quarter (w >> 1) of d.
// us: [B][d] bf16 scratch in shared memory.
// This warp's chunk of its router row (d <= 4096: <= 4 x 16 B per lane),
// loaded by the gate CTAs BEFORE the programmatic-dependency wait: the router
// weights do not depend on the previous layer, so the load overlaps its FFN's
// tail (gate_decide_kernel).
constexpr uint32_t kGateWPre = 4;
struct GateWPre {
  uint4 w[kGateWPre];
  bool ok;
};
__device__ __forceinline__ GateWPre gate_w_prefetch(const GateArgs& a, uint32_t gi) {
  GateWPre r;
  const int lane = lane_id(), warp = warp_id();
  const uint32_t rows = a.E + (a.wsg ? 1u : 0u), row = 2 * gi + (warp & 1), q = warp >> 1;
  const uint32_t per_q = a.d / 32, c0 = q * per_q;  // (d / 8) / 4 vectors per quarter
  r.ok = row < rows && per_q % 32 == 0 && per_q / 32 <= kGateWPre;
  if (r.ok) {
    const uint4* wv = reinterpret_cast<const uint4*>(row < a.E ? a.wg + (size_t)row * a.d : a.wsg);
#pragma unroll
    for (uint32_t j = 0; j < kGateWPre; ++j)
      if (j < per_q / 32) r.w[j] = __ldg(wv + c0 + j * 32 + lane);
  }
  return r;
}

__device__ inline void gate_phase(const GateArgs& a, uint16_t* us, uint32_t gi, uint32_t ng, const uint16_t* xsrc,
                                  float* logits_out, bool write_u, const GateWPre* wp = nullptr) {
  __shared__ float part[4][2][kMaxB];
  __shared__ float inv_rms[kMaxB];
  const int lane = lane_id(), warp = warp_id();
  const uint32_t d = a.d, B = a.B;
  const uint32_t nvec = d / 8;
  // x -> shared memory once, 8 independent 16 B loads in flight per thread
  // (a strided one-load-per-iteration loop is L2-latency-bound at B = 32)
  {
    const uint32_t n = B * nvec;
    const uint4* xg = reinterpret_cast<const uint4*>(xsrc);
    uint4* xs = reinterpret_cast<uint4*>(us);
    for (uint32_t i0 = threadIdx.x; i0 < n; i0 += 8 * blockDim.x) {
      uint4 v[8];
#pragma unroll
      for (uint32_t j = 0; j < 8; ++j) {
        const uint32_t i = i0 + j * blockDim.x;
        if (i < n) v[j] = xg[i];
      }
#pragma unroll
      for (uint32_t j = 0; j < 8; ++j) {
        const uint32_t i = i0 + j * blockDim.x;
        if (i < n) xs[i] = v[j];
      }
    }
  }
  __syncthreads();
  // RMSNorm (eps 1e-6, unit weight): one warp per token
  for (uint32_t t = warp; t < B; t += kGateThreads / 32) {
    const uint4* xv = reinterpret_cast<const uint4*>(us + (size_t)t * d);
    float ss = 0.f;
    for (uint32_t c = lane; c < nvec; c += 32) {
      const uint4 v = xv[c];
      ss += dot8(v, v);
    }
    ss = warp_sum(ss);
    if (lane == 0) inv_rms[t] = __frsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)d), 1e-6f));
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < B * nvec; i += blockDim.x) {
    const uint32_t t = i / nvec, c = i % nvec;
    const uint4 v = reinterpret_cast<const uint4*>(us + (size_t)t * d)[c];
    const float r = inv_rms[t];
    const uint32_t in[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float lo = __fmul_rn(__uint_as_float(in[j] << 16), r);
      const float hi = __fmul_rn(__uint_as_float(in[j] & 0xffff0000u), r);
      uint32_t bl = __float_as_uint(lo), bh = __float_as_uint(hi);
      bl += 0x7FFFu + ((bl >> 16) & 1u);
      bh += 0x7FFFu + ((bh >> 16) & 1u);
      o[j] = (bl >> 16) | (bh & 0xffff0000u);
    }
    const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
    reinterpret_cast<uint4*>(us + (size_t)t * d)[c] = ov;
    if (write_u && gi == 0) reinterpret_cast<uint4*>(a.u + (size_t)t * d)[c] = ov;
    if (write_u && a.ut && gi == (ng > 1 ? 1u : 0u)) {
      // 16 B chunk (c % 8) of K-block c / 8, row t: chunk position (c ^ t) % 8
      const uint32_t off = (c >> 3) * a.ut_rows * 128u + (t >> 3) * 1024u + (t & 7u) * 128u + (((c ^ t) & 7u) << 4);
      *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(a.ut) + off) = ov;
    }
  }
  __syncthreads();
  const uint32_t rows = a.E + (a.wsg ? 1u : 0u);
  const uint32_t row = 2 * gi + (warp & 1);
  const uint32_t q = warp >> 1;
  if (row < rows) {
    const uint16_t* w = row < a.E ? a.wg + (size_t)row * d : a.wsg;
    const uint4* wv = reinterpret_cast<const uint4*>(w);
    const uint32_t c0 = q * (nvec / 4), c1 = (q + 1) * (nvec / 4);
    if (B <= 4 || nvec / 4 != 64) {
      for (uint32_t t = 0; t < B; ++t) {
        const uint4* uv = reinterpret_cast<const uint4*>(us + (size_t)t * d);
        float s = 0.f;
        if (wp && wp->ok) {  // same order as the loop below: c = c0 + lane + 32 j
#pragma unroll
          for (uint32_t j = 0; j < kGateWPre; ++j)
            if (j < nvec / 4 / 32) s += dot8(wp->w[j], uv[c0 + j * 32 + lane]);
        } else {
          for (uint32_t c = c0 + lane; c < c1; c += 32) s += dot8(__ldg(wv + c), uv[c]);
        }
        s = warp_sum(s);
        if (lane == 0) part[q][warp & 1][t] = s;
      }
    } else {
      // d = 2048: the lane's two weight vectors stay in registers; per-lane
      // partial dots of all tokens, then one transposed butterfly (31
      // shuffles for 32 tokens instead of 5 per token): lane t ends with
      // token t's sum
      const bool pre = wp && wp->ok;
      const uint4 w0 = pre ? wp->w[0] : __ldg(wv + c0 + lane), w1 = pre ? wp->w[1] : __ldg(wv + c0 + 32 + lane);
      float p[32];
#pragma unroll
      for (uint32_t t = 0; t < 32; ++t) {
        p[t] = 0.f;
        if (t < B) {
          const uint4* uv = reinterpret_cast<const uint4*>(us + (size_t)t * d);
          p[t] = dot8(w0, uv[c0 + lane]) + dot8(w1, uv[c0 + 32 + lane]);
        }
      }
#pragma unroll
      for (uint32_t o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (uint32_t i = 0; i < o; ++i) {
          const float send = up ? p[i] : p[i + o];
          const float keep = up ? p[i + o] : p[i];
          p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if ((uint32_t)lane < B) part[q][warp & 1][lane] = p[0];
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * B) {
    const uint32_t r = threadIdx.x & 1, t = threadIdx.x >> 1;
    const uint32_t rr = 2 * gi + r;
    if (rr < rows) {
      const float s = ((part[0][r][t] + part[1][r][t]) + part[2][r][t]) + part[3][r][t];
      logits_out[(size_t)t * (a.E + 1) + rr] = s;
    }
  }
}

// ------------------------------------------------------------------- FFN
struct FfnArgs {
  const Plan* plan;
  const uint16_t* u;       // [B][d]
  const uint16_t* x_in;    // [B][d]
  uint16_t* x_out;         // [B][d]
  float* y_out;            // [B][d] fp32 MoE output of this layer
  float* h;                // [kMaxItems][B][Fmax]
  uint32_t* ctr;           // [0,kMaxItems) item gate_up done, [kMaxItems] d2d barrier, [kMaxItems+1] exit
  const uint32_t* copies_done;
  uint32_t* ffn_done;
  uint32_t B, d, Fmax;
  uint32_t rows_per_warp;  // ceil(d / total warps)
};

__device__ __forceinline__ void wait_copy(const uint32_t* copies_done, uint32_t id) {
  if (id == 0) return;
  if (threadIdx.x == 0) {
    const uint64_t t0 = globaltimer_ns();
    while ((int32_t)(ld_acquire_u32(copies_done) - id) < 0) {
      __nanosleep(256);
      if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 1u); break; }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void signal_item(uint32_t* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
  }
}

__device__ __forceinline__ void wait_item(const uint32_t* ctr, uint32_t target) {
  if (threadIdx.x == 0) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_u32(ctr) < target) {
      __nanosleep(64);
      if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 2u); break; }
    }
  }
  __syncthreads();
}

// gate_up for one item over this CTA's share of rows (rows strided by warps).
template <int NT>
__device__ inline void gate_up_rows(const Item& it, const uint16_t* us, uint32_t d, float* h_item,
                                    uint32_t Fmax, uint32_t gw, uint32_t nW) {
  const int lane = lane_id();
  const uint32_t F = it.F, n = it.n_tok;
  const uint32_t nvec = d / 8;
  constexpr int UNR = NT >= 16 ? 2 : (NT >= 8 ? 4 : 8);
  for (uint32_t r = gw; r < F; r += nW) {
    const uint4* G = reinterpret_cast<const uint4*>(it.w + (size_t)r * d);
    const uint4* U = reinterpret_cast<const uint4*>(it.w + ((size_t)F + r) * d);
    float ag[NT], au[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) { ag[t] = 0.f; au[t] = 0.f; }
    for (uint32_t c0 = lane; c0 < nvec; c0 += 32 * UNR) {
      uint4 g[UNR], uu[UNR];
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const uint32_t c = c0 + 32 * j;
        if (c < nvec) { g[j] = ldg_cg(G + c); uu[j] = ldg_cg(U + c); }
      }
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const uint32_t c = c0 + 32 * j;
        if (c < nvec) {
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if ((uint32_t)t < n) {
              const uint4 xv = reinterpret_cast<const uint4*>(us + (size_t)it.tok[t] * d)[c];
              ag[t] += dot8(g[j], xv);
              au[t] += dot8(uu[j], xv);
            }
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      if ((uint32_t)t < n) {
        const float gs = warp_sum(ag[t]);
        const float us2 = warp_sum(au[t]);
        if (lane == (t & 31)) {
          const float silu = __fdiv_rn(gs, 1.0f + expf(-gs));
          h_item[(size_t)t * Fmax + r] = silu * us2;
        }
      }
    }
  }
}

// down projection of one item accumulated into this warp's output rows.
template <int NT>
__device__ inline void down_rows(const Item& it, uint32_t d, const float* h_item, uint32_t Fmax,
                                 uint32_t gw, uint32_t nW, uint32_t rpw, float* acc /*[rpw][kMaxB]*/) {
  const int lane = lane_id();
  const uint32_t F = it.F, n = it.n_tok;
  const uint32_t nvec = F / 8;
  const uint16_t* Wd = it.w + 2 * (size_t)F * d;
  for (uint32_t m = 0; m < rpw; ++m) {
    const uint32_t o = gw + m * nW;
    if (o >= d) break;
    const uint4* D = reinterpret_cast<const uint4*>(Wd + (size_t)o * F);
    float a[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) a[t] = 0.f;
    constexpr int UNR = NT >= 16 ? 2 : 4;
    for (uint32_t c0 = lane; c0 < nvec; c0 += 32 * UNR) {
      uint4 wv[UNR];
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const uint32_t c = c0 + 32 * j;
        if (c < nvec) wv[j] = ldg_cg(D + c);
      }
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const uint32_t c = c0 + 32 * j;
        if (c < nvec) {
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if ((uint32_t)t < n) {
              const float4* hp = reinterpret_cast<const float4*>(h_item + (size_t)t * Fmax + c * 8);
              a[t] += dot8f(wv[j], hp[0], hp[1]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      if ((uint32_t)t < n) {
        const float s = warp_sum(a[t]);
        if (lane == 0) {
          const uint32_t tok = it.tok[t];
          acc[m * kMaxB + tok] = fmaf(it.wt[t], s, acc[m * kMaxB + tok]);
        }
      }
    }
  }
}

template <int NT>
__device__ inline void item_gate_up(const Plan* p, uint32_t i, const uint16_t* us, const FfnArgs& a,
                                    uint32_t gw, uint32_t nW) {
  gate_up_rows<NT>(p->items[i], us, a.d, a.h + (size_t)i * kMaxB * a.Fmax, a.Fmax, gw, nW);
}

template <int NTMAX>
__device__ inline void dispatch_gate_up(const Plan* p, uint32_t i, const uint16_t* us, const FfnArgs& a,
                                        uint32_t gw, uint32_t nW) {
  const uint32_t n = p->items[i].n_tok;
  if (NTMAX == 1 || n <= 1) item_gate_up<1>(p, i, us, a, gw, nW);
  else if (NTMAX == 2 || n <= 2) item_gate_up<(NTMAX < 2 ? NTMAX : 2)>(p, i, us, a, gw, nW);
  else if (NTMAX == 4 || n <= 4) item_gate_up<(NTMAX < 4 ? NTMAX : 4)>(p, i, us, a, gw, nW);
  else if (NTMAX == 8 || n <= 8) item_gate_up<(NTMAX < 8 ? NTMAX : 8)>(p, i, us, a, gw, nW);
  else if (NTMAX == 16 || n <= 16) item_gate_up<(NTMAX < 16 ? NTMAX : 16)>(p, i, us, a, gw, nW);
  else item_gate_up<NTMAX>(p, i, us, a, gw, nW);
}

template <int NT>
__device__ inline void item_down(const Plan* p, uint32_t i, const FfnArgs& a, uint32_t gw, uint32_t nW,
                                 float* acc) {
  down_rows<NT>(p->items[i], a.d, a.h + (size_t)i * kMaxB * a.Fmax, a.Fmax, gw, nW, a.rows_per_warp, acc);
}

template <int NTMAX>
__device__ inline void dispatch_down(const Plan* p, uint32_t i, const FfnArgs& a, uint32_t gw,
                                     uint32_t nW, float* acc) {
  const uint32_t n = p->items[i].n_tok;
  if (NTMAX == 1 || n <= 1) item_down<1>(p, i, a, gw, nW, acc);
  else if (NTMAX == 2 || n <= 2) item_down<(NTMAX < 2 ? NTMAX : 2)>(p, i, a, gw, nW, acc);
  else if (NTMAX == 4 || n <= 4) item_down<(NTMAX < 4 ? NTMAX : 4)>(p, i, a, gw, nW, acc);
  else if (NTMAX == 8 || n <= 8) item_down<(NTMAX < 8 ? NTMAX : 8)>(p, i, a, gw, nW, acc);
  else if (NTMAX == 16 || n <= 16) item_down<(NTMAX < 16 ? NTMAX : 16)>(p, i, a, gw, nW, acc);
  else item_down<NTMAX>(p, i, a, gw, nW, acc);
}

constexpr int kMaxRowsPerWarp = 4;

template <int NTMAX>
__global__ void __launch_bounds__(kFfnThreads, 1) ffn_kernel(FfnArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint16_t* us = reinterpret_cast<uint16_t*>(smem_raw);  // [B][d]
  __shared__ float acc_s[kFfnWarps][kMaxRowsPerWarp * kMaxB];
  const Plan* p = a.plan;
  const int lane = lane_id(), warp = warp_id();
  const uint32_t nW = gridDim.x * kFfnWarps;
  const uint32_t gw = blockIdx.x * kFfnWarps + warp;
  const uint32_t nvec = a.d / 8;
  for (uint32_t i = threadIdx.x; i < a.B * nvec; i += blockDim.x)
    reinterpret_cast<uint4*>(us)[i] = reinterpret_cast<const uint4*>(a.u)[i];
  float* acc = acc_s[warp];
  for (uint32_t i = lane; i < kMaxRowsPerWarp * kMaxB; i += 32) acc[i] = 0.f;
  __syncthreads();

  const uint32_t n_items = p->n_items, n_ready = p->n_ready;
  // phase 1: gate_up of every ready item
  for (uint32_t i = 0; i < n_ready; ++i) {
    dispatch_gate_up<NTMAX>(p, i, us, a, gw, nW);
    signal_item(&a.ctr[i]);
  }
  // phase 2: down of the ready items (overlaps in-flight uploads)
  for (uint32_t i = 0; i < n_ready; ++i) {
    wait_item(&a.ctr[i], gridDim.x);
    dispatch_down<NTMAX>(p, i, a, gw, nW, acc);
    __syncwarp();
  }
  // phase 3: items gated on uploads, in upload order
  for (uint32_t i = n_ready; i < n_items; ++i) {
    wait_copy(a.copies_done, p->items[i].wait);
    dispatch_gate_up<NTMAX>(p, i, us, a, gw, nW);
    signal_item(&a.ctr[i]);
    wait_item(&a.ctr[i], gridDim.x);
    dispatch_down<NTMAX>(p, i, a, gw, nW, acc);
    __syncwarp();
  }
  // epilogue: residual add, bf16 hidden for the next layer, fp32 MoE output
  for (uint32_t m = 0; m < a.rows_per_warp; ++m) {
    const uint32_t o = gw + m * nW;
    if (o >= a.d) break;
    for (uint32_t t = lane; t < a.B; t += 32) {
      const float y = acc[m * kMaxB + t];
      const float xo = bf2f(a.x_in[(size_t)t * a.d + o]) + y;
      a.x_out[(size_t)t * a.d + o] = f32_to_bf16_rne(xo);
      a.y_out[(size_t)t * a.d + o] = y;
    }
  }
  // deferred admissions: staging -> slot once every CTA finished reading
  if (p->n_d2d) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&a.ctr[kMaxItems], 1u);
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_u32(&a.ctr[kMaxItems]) < gridDim.x) {
        __nanosleep(128);
        if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 3u); break; }
      }
    }
    __syncthreads();
    const uint64_t nv = p->d2d_elems / 8;
    for (uint32_t j = 0; j < p->n_d2d; ++j) {
      const uint4* src = reinterpret_cast<const uint4*>(p->d2d[j].src);
      uint4* dst = reinterpret_cast<uint4*>(p->d2d[j].dst);
      for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv;
           v += (uint64_t)gridDim.x * blockDim.x)
        dst[v] = ldg_cg(src + v);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(&a.ctr[kMaxItems + 1], 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.ffn_done), "r"(p->seq) : "memory");
    }
  }
}

}  // namespace moeb
