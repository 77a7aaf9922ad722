// ffn_umma.cuh — batched-decode (B = 2..32) grouped SwiGLU FFN on the 5th-gen
// tensor cores (tcgen05.mma, accumulators in TMEM, operands staged in shared
// memory by cp.async.bulk), sm_100a.
//
// Why tensor cores here and not at B = 1: with B tokens per step an expert's
// weight tile is multiplied by up to B activation vectors, a [128 x K] x
// [K x N] contraction with N = the batch. It is still HBM-bound (every weight
// byte is read once per step), so the MMA computes ALL B token columns for
// every expert — tokens not routed to an expert get a zero combine weight in
// the epilogue — which removes every gather/scatter and keeps one B operand
// (the batch's activations) for all experts.
//
// Weights are stored "UMMA-tiled" (weights.cuh synth_tiled_kernel): every
// 16 KB block is a [128 rows x 64 K] bf16 tile already in the canonical
// SWIZZLE_128B K-major layout the MMA reads, so one 1-D bulk copy per stage
// lands a ready operand (no tensor maps: the expert pointer comes from the
// device-side plan, slot or staging buffer alike).
//   gate_up section: unit u (128 intermediate rows) x K-block kb (64 of d):
//                    [gate tile 16 KB][up tile 16 KB]
//   down section:    unit m (128 output rows) x K-pair kp (128 of F):
//                    [down tile kb = 2kp][down tile kb = 2kp + 1]
//
// Work units (grid-dynamic, one atomic grab per unit):
//   gate_up (item, u): 32 KB stages over d/64 K-blocks; two accumulators
//     (gate, up: N = Nx columns each); the epilogue thread of TMEM lane j owns
//     intermediate row j of the unit: h = silu(g) * up for every
//     token column, split into bf16 hi + lo (h = hi + lo to 2^-17), stored as
//     the down pass's B operand ([K-block][2 Bp rows][128 B], SW128).
//   down (item, m): 32 KB weight stage + the item's h K-pair (from L2), one
//     accumulator of N = 2 Bp columns (hi rows, lo rows); the epilogue writes
//     the item's partial w_tok * (hi + lo) to part[item, split].
// A down unit waits for its item's gate_up units (per-item grid counter).
// Items whose weights are still on the PCIe copy stream are gated on
// copies_done by the producer. End: grid barrier, each CTA sums its output
// rows over the items in plan order (deterministic: no atomics on data),
// residual, bf16 hidden for the next layer.
//
// Roles: warp 0 producer (one lane), warp 1 TMEM owner + MMA issuer (one
// lane), warps 2..5 epilogue (TMEM lane quadrant = warp % 4).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "ffn_tma.cuh"

namespace moeb {

constexpr uint32_t kUmBlk = 16384;          // one [128 x 64] bf16 tile
constexpr uint32_t kUmA = 2 * kUmBlk;       // weight bytes per stage
constexpr uint32_t kUmRec = 4;              // unit records in flight
constexpr uint32_t kUmMaxStages = 8;
constexpr uint32_t kUmThreads = 6 * 32;
constexpr uint32_t kUmTmemCols = 128;       // two accumulator buffers of <= 64 columns
// grid counter reused from the speculative kernel (B > 1 has no speculative
// phase): CTAs done with their units
constexpr int kUmDoneCtr = kFfnSpecDoneCtr;

struct UmArgs {
  FfnTArgs f;
  uint16_t* xt;     // activations, SW128-tiled: [d/64][Nx][64] bf16 (written by the gate phase)
  float* part;      // partial outputs [item, down split][B][d] fp32
  float* gpart;     // gate_up K-split partials [tile][split][2 Nx][128] fp32
  uint32_t* gcnt;   // per-tile split arrivals (monotonic: +KS per tile per launch)
  uint32_t KS;      // gate_up K-splits (divides d/64)
  uint32_t dn_st;   // K-pair stages per down unit
  uint32_t Nx;      // token rows of the gate_up B operand (multiple of 16)
  uint32_t Bp;      // token rows of each hi / lo half of the down B operand (multiple of 8)
  uint32_t stages;
  uint32_t stage_bytes;
};

// ------------------------------------------------------------ tcgen05 PTX
__device__ __forceinline__ uint64_t um_desc(uint32_t saddr) {
  // SWIZZLE_128B K-major: SBO = 1024 B (8-row groups), LBO unused (1),
  // descriptor version 1 (sm_100), layout type 2 (128 B swizzle)
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: bf16 A/B, fp32 D, both K-major, M = 128
__host__ __device__ constexpr uint32_t um_idesc(uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void um_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void um_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void um_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void um_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void um_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void um_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// store kept in L2 (evict_last): the down partials are read back by the
// final sum after the rest of the weight stream has passed through L2
__device__ __forceinline__ void st_keep(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void um_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void wait_ctr_ge(const uint32_t* p, uint32_t v, uint32_t code) {
  const uint64_t t0 = globaltimer_ns();
  while (ld_acquire_u32(p) < v) {
    __nanosleep(32);
    if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, code); break; }
  }
}
// byte offset of element (r, k) of a [rows x 64] bf16 SW128 K-major tile
__host__ __device__ __forceinline__ uint32_t sw128_off(uint32_t r, uint32_t k) {
  return (r >> 3) * 1024u + (r & 7u) * 128u + ((((k >> 3) ^ r) & 7u) << 4) + (k & 7u) * 2u;
}

struct UmRec {
  uint32_t kind;   // 0 gate_up, 1 down, 2 end
  uint32_t item;
  uint32_t idx;    // gate_up tile u / down row tile m
  uint32_t split;  // gate_up K-split / down K-split
  uint32_t s0;     // first K-block (gate_up) / K-pair (down) of the unit
  uint32_t n_st;   // stages of the unit
};

__global__ void __launch_bounds__(kUmThreads, 1) ffn_umma_kernel(const __grid_constant__ UmArgs ua) {
  const FfnTArgs& a = ua.f;
  extern __shared__ unsigned char um_smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kUmMaxStages], empty_bar[kUmMaxStages];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ __align__(8) uint64_t rfull_bar[kUmRec], rempty_bar[kUmRec];
  __shared__ UmRec recs[kUmRec];
  __shared__ uint32_t s_tmem;
  // per item (plan order): first gate_up unit, first down unit, first tile,
  // first down partial
  __shared__ uint32_t s_gu0[kMaxItems + 1], s_dn0[kMaxItems + 1], s_tb[kMaxItems + 1], s_pb[kMaxItems + 1];
  __shared__ uint32_t s_ngu[kMaxItems + 1], s_ndn[kMaxItems + 1];
  __shared__ uint32_t s_ni, s_last;
  __shared__ uint32_t s_F[kMaxItems], s_wait[kMaxItems];
  __shared__ const unsigned char* s_w[kMaxItems];

  asm volatile("griddepcontrol.launch_dependents;");
  if (a.tl && blockIdx.x == 0 && threadIdx.x == 0) a.tl[7] = globaltimer_ns();
  const uint32_t G = gridDim.x, c = blockIdx.x;
  const uint32_t d = a.d, B = a.B, S = ua.stages, SB = ua.stage_bytes, Nx = ua.Nx, Bp = ua.Bp, Ndn = 2 * Bp;
  const int warp = warp_id(), lane = lane_id();
  // 1 KB-aligned ring (the SW128 atoms need it)
  const uint32_t raw_addr = smem_u32(um_smem_raw);
  unsigned char* ring = um_smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  const uint32_t ring_addr = smem_u32(ring);
  float* s_wv = reinterpret_cast<float*>(ring + (size_t)S * SB);  // [item][B] combine weight per token column
  const uint32_t nkb = d / 64, nm = d / 128, KS = ua.KS, kst = nkb / ua.KS, dn_st = ua.dn_st;

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < S; ++s) {
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
                 "n"(kUmTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    um_fence_before();
  }
  __syncthreads();  // barriers initialised, TMEM allocated
  um_fence_after();
  const uint32_t tmem = s_tmem;
  // Speculative start (the decide kernel publishes the shared expert and
  // the experts certain to be selected right after classification): their
  // gate_up units run while the decision finishes — gate_up does not depend
  // on the token lists (every token column is computed; the combine weights
  // are applied per column in the down epilogue). The final plan lists them
  // first, in the same order, and is taken from the decide kernel's release
  // flag. Without a speculative plan: PDL wait for the decide kernel.
  // (Running the speculative items' down units early as well, with the
  // weights moved to the final sum, measured no faster in the pipeline and
  // slower standalone.)
  const bool spec = a.spec_plan != nullptr;
  if (!spec) asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // warp 0 stages the item tables (all lanes); lane 0 streams the units
    const uint64_t pol = l2_evict_first_policy(), pol_keep = l2_evict_last_policy();
    uint32_t k = 0, u = 0;  // ring step, unit record count
    auto load_items = [&](const Plan* pl, uint32_t i0, uint32_t i1) {
      for (uint32_t i = i0 + lane; i < i1; i += 32) {
        s_F[i] = __ldcg(&pl->items[i].F);
        s_wait[i] = __ldcg(&pl->items[i].wait);
        s_w[i] = reinterpret_cast<const unsigned char*>(
            __ldcg(reinterpret_cast<const unsigned long long*>(&pl->items[i].w)));
      }
    };
    // unit tables of items [0, ni): gate_up units of items >= g0, down
    // units unless gu_only
    auto build = [&](uint32_t ni, uint32_t nr, uint32_t g0, bool gu_only) -> uint32_t {
      uint32_t tb = 0, pb = 0;
      for (uint32_t i = 0; i < ni; ++i) {
        s_tb[i] = tb;
        s_pb[i] = pb;
        const uint32_t t = s_F[i] / 128;
        tb += t;
        pb += (t + dn_st - 1) / dn_st;
      }
      s_tb[ni] = tb;
      s_pb[ni] = pb;
      uint32_t acc = 0;
      // [gate_up of the ready items][down of the ready items], then per
      // waiting item [gate_up][down]
      for (uint32_t i = 0; i < nr; ++i) {
        s_gu0[i] = acc;
        s_ngu[i] = i >= g0 ? (s_tb[i + 1] - s_tb[i]) * KS : 0u;
        acc += s_ngu[i];
      }
      for (uint32_t i = 0; i < nr; ++i) {
        s_dn0[i] = acc;
        s_ndn[i] = gu_only ? 0u : nm * (s_pb[i + 1] - s_pb[i]);
        acc += s_ndn[i];
      }
      for (uint32_t i = nr; i < ni; ++i) {
        s_gu0[i] = acc;
        s_ngu[i] = (s_tb[i + 1] - s_tb[i]) * KS;
        acc += s_ngu[i];
        s_dn0[i] = acc;
        s_ndn[i] = nm * (s_pb[i + 1] - s_pb[i]);
        acc += s_ndn[i];
      }
      return acc;
    };
    auto publish = [&](const UmRec& r) {
      const uint32_t j = u % kUmRec;
      mbar_wait(&rempty_bar[j], ((u / kUmRec) & 1) ^ 1);
      recs[j] = r;
      mbar_arrive(&rfull_bar[j]);
      ++u;
    };
    // units [0, total) of the current tables, grabbed from counter ctr_i
    auto run_units = [&](uint32_t ctr_i, uint32_t total, uint32_t ni) {
      uint32_t nxt = atomicAdd(&a.ctr[ctr_i], 1u);
      while (nxt < total) {
        const uint32_t unit = nxt;
        nxt = atomicAdd(&a.ctr[ctr_i], 1u);
        UmRec r{2u, 0u, 0u, 0u, 0u, 0u};
        for (uint32_t i = 0; i < ni; ++i) {
          if (unit - s_gu0[i] < s_ngu[i]) {
            const uint32_t q = unit - s_gu0[i];
            r = UmRec{0u, i, q / KS, q % KS, (q % KS) * kst, kst};
            break;
          }
          if (unit - s_dn0[i] < s_ndn[i]) {
            const uint32_t tiles = s_tb[i + 1] - s_tb[i], DS = s_pb[i + 1] - s_pb[i];
            const uint32_t q = unit - s_dn0[i], ds = q % DS;
            r = UmRec{1u, i, q / DS, ds, ds * dn_st, min(dn_st, tiles - ds * dn_st)};
            break;
          }
        }
        publish(r);
        const uint32_t F = s_F[r.item], wait_id = s_wait[r.item];
        if (wait_id) {
          const uint64_t t0 = globaltimer_ns();
          while ((int32_t)(ld_acquire_u32(a.copies_done) - wait_id) < 0) {
            __nanosleep(128);
            if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 1u); break; }
          }
          if (a.tl && c == 0) a.tl[1] = globaltimer_ns();
          fence_proxy_async_global();
        }
        const unsigned char* w = s_w[r.item];
        if (r.kind == 0) {
          const unsigned char* src = w + ((size_t)r.idx * nkb + r.s0) * kUmA;
          const uint32_t xb = Nx * 128;
          const unsigned char* xs = reinterpret_cast<const unsigned char*>(ua.xt) + (size_t)r.s0 * xb;
          for (uint32_t s = 0; s < r.n_st; ++s, ++k) {
            const uint32_t st = k % S;
            mbar_wait(&empty_bar[st], ((k / S) & 1) ^ 1);
            mbar_expect_tx(&full_bar[st], kUmA + xb);
            bulk_g2s(ring + st * SB, src + (size_t)s * kUmA, kUmA, &full_bar[st], pol);
            bulk_g2s(ring + st * SB + kUmA, xs + (size_t)s * xb, xb, &full_bar[st], pol_keep);
          }
        } else {
          // h of the item: every gate_up unit must have landed
          wait_ctr_ge(&a.ctr[r.item], F / 128, 8u);
          if (a.tl) atomicCAS(reinterpret_cast<unsigned long long*>(a.tl + 10), 0ull, (unsigned long long)globaltimer_ns());
          fence_proxy_async_global();
          const unsigned char* src = w + 2 * (size_t)F * d * 2 + ((size_t)r.idx * (F / 128) + r.s0) * kUmA;
          const uint32_t hb = 2 * Ndn * 128;
          const unsigned char* hs =
              reinterpret_cast<const unsigned char*>(a.h + (size_t)r.item * kMaxB * a.Fmax) + (size_t)r.s0 * hb;
          for (uint32_t s = 0; s < r.n_st; ++s, ++k) {
            const uint32_t st = k % S;
            mbar_wait(&empty_bar[st], ((k / S) & 1) ^ 1);
            mbar_expect_tx(&full_bar[st], kUmA + hb);
            bulk_g2s(ring + st * SB, src + (size_t)s * kUmA, kUmA, &full_bar[st], pol);
            bulk_g2s(ring + st * SB + kUmA, hs + (size_t)s * hb, hb, &full_bar[st], pol_keep);
          }
        }
      }
    };
    uint32_t n_spec = 0;
    if (spec) {
      if (lane == 0) {
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_u32(a.spec_flag) != a.seq) {
          __nanosleep(64);
          if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 5u); break; }
        }
        if (a.tl && c == 0) a.tl[6] = globaltimer_ns();
      }
      __syncwarp();
      n_spec = ld_acquire_u32(&a.spec_plan->n_spec);
      load_items(a.spec_plan, 0, n_spec);
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async_global();  // the activation tiles (gate phase) are read by bulk copies
        const uint32_t tot = build(n_spec, n_spec, 0, true);
        run_units(kFfnSpecGuCtr, tot, n_spec);
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_u32(a.spec_flag + 1) != a.seq) {
          __nanosleep(32);
          if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 6u); break; }
        }
      }
      __syncwarp();
    }
    // the final plan: items, and each item's combine weight per token column
    const uint32_t ni = ld_acquire_u32(&a.plan->n_items), nr = __ldcg(&a.plan->n_ready);
    load_items(a.plan, n_spec, ni);
    for (uint32_t i = lane; i < ni * B; i += 32) s_wv[i] = 0.f;
    __syncwarp();
    for (uint32_t i = lane; i < ni * kMaxB; i += 32) {
      const Item& it = a.plan->items[i / kMaxB];
      const uint32_t jt = i % kMaxB;
      if (jt < __ldcg(&it.n_tok)) s_wv[(i / kMaxB) * B + __ldcg(&it.tok[jt])] = __ldcg(&it.wt[jt]);
    }
    __syncwarp();
    if (lane == 0) {
      if (a.tl && c == 0) a.tl[0] = globaltimer_ns();
      fence_proxy_async_global();
      const uint32_t tot = build(ni, nr, n_spec, false);
      s_ni = ni;
      run_units(kFfnGuCtr, tot, ni);
      publish(UmRec{2u, 0u, 0u, 0u, 0u, 0u});
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t id_gu = um_idesc(Nx), id_dn = um_idesc(Ndn);
      uint32_t k = 0;
      for (uint32_t u = 0;; ++u) {
        const uint32_t j = u % kUmRec;
        mbar_wait(&rfull_bar[j], (u / kUmRec) & 1);
        const UmRec r = recs[j];
        if (r.kind == 2) break;
        const uint32_t b = u & 1;
        mbar_wait(&tempty_bar[b], ((u >> 1) & 1) ^ 1);
        um_fence_after();
        const uint32_t acc0 = tmem + b * 64;
        const uint32_t n_st = r.n_st;
        for (uint32_t s = 0; s < n_st; ++s, ++k) {
          const uint32_t st = k % S;
          mbar_wait(&full_bar[st], (k / S) & 1);
          um_fence_after();
          const uint32_t sa = ring_addr + st * SB;
          if (r.kind == 0) {
#pragma unroll
            for (uint32_t kk = 0; kk < 4; ++kk) {
              const uint64_t bx = um_desc(sa + kUmA + kk * 32);
              um_mma(acc0, um_desc(sa + kk * 32), bx, id_gu, (s | kk) != 0);
              um_mma(acc0 + Nx, um_desc(sa + kUmBlk + kk * 32), bx, id_gu, (s | kk) != 0);
            }
          } else {
#pragma unroll
            for (uint32_t hf = 0; hf < 2; ++hf)
#pragma unroll
              for (uint32_t kk = 0; kk < 4; ++kk)
                um_mma(acc0, um_desc(sa + hf * kUmBlk + kk * 32), um_desc(sa + kUmA + hf * Ndn * 128 + kk * 32),
                       id_dn, (s | hf | kk) != 0);
          }
          um_commit(&empty_bar[st]);  // frees the stage once these MMAs have read it
        }
        um_commit(&tfull_bar[b]);
      }
    }
  } else {
    // ------------------------------------------------------------- epilogue
    const uint32_t q = warp & 3;  // TMEM lane quadrant this warp may access
    const uint64_t pol_part = l2_evict_last_policy();
    const uint32_t et = (warp - 2) * 32 + lane;
    for (uint32_t u = 0;; ++u) {
      const uint32_t j = u % kUmRec;
      mbar_wait(&rfull_bar[j], (u / kUmRec) & 1);
      const UmRec r = recs[j];
      if (r.kind == 2) break;
      const uint32_t b = u & 1;
      mbar_wait(&tfull_bar[b], (u >> 1) & 1);
      um_fence_after();
      const uint32_t ta = tmem + ((q * 32) << 16) + b * 64;
      if (r.kind == 0) {
        float g[32], up[32];
        um_ld16(ta, g);
        um_ld16(ta + Nx, up);
        if (Nx > 16) {
          um_ld16(ta + 16, g + 16);
          um_ld16(ta + Nx + 16, up + 16);
        }
        um_ld_wait();
        um_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[b]);
        if (KS > 1) {
          // K-split: publish this split's partial dots; the last split of
          // the tile sums all of them in split order (deterministic)
          const uint32_t T = s_tb[r.item] + r.idx;
          float* gp = ua.gpart + (size_t)T * KS * 2 * Nx * 128 + q * 32 + lane;
          float* mine = gp + (size_t)r.split * 2 * Nx * 128;
#pragma unroll
          for (uint32_t n = 0; n < 32; ++n) {
            if (n >= Nx) break;
            __stcg(mine + n * 128, g[n]);
            __stcg(mine + (Nx + n) * 128, up[n]);
          }
          __threadfence();
          asm volatile("bar.sync 2, 128;" ::: "memory");
          if (et == 0) s_last = (atomicAdd(&ua.gcnt[T], 1u) + 1) % KS == 0;
          asm volatile("bar.sync 2, 128;" ::: "memory");
          if (!s_last) {
            if (et == 0) mbar_arrive(&rempty_bar[j]);
            continue;
          }
          __threadfence();
          // every split's 2 Nx values in flight at once, summed in split order
#pragma unroll
          for (uint32_t n = 0; n < 32; ++n) g[n] = up[n] = 0.f;
          for (uint32_t ks = 0; ks < KS; ++ks) {
            const float* src = gp + (size_t)ks * 2 * Nx * 128;
#pragma unroll
            for (uint32_t n0 = 0; n0 < 32; n0 += 16) {
              if (n0 >= Nx) break;
              float tg[16], tu[16];
#pragma unroll
              for (uint32_t n = 0; n < 16; ++n) {
                tg[n] = __ldcg(src + (n0 + n) * 128);
                tu[n] = __ldcg(src + (Nx + n0 + n) * 128);
              }
#pragma unroll
              for (uint32_t n = 0; n < 16; ++n) {
                g[n0 + n] += tg[n];
                up[n0 + n] += tu[n];
              }
            }
          }
        }
        // intermediate row jr of the item -> down K-block jr / 64, column jr % 64
        const uint32_t jr = r.idx * 128 + q * 32 + lane;
        unsigned char* hb = reinterpret_cast<unsigned char*>(a.h + (size_t)r.item * kMaxB * a.Fmax) +
                            (size_t)(jr >> 6) * Ndn * 128;
        const uint32_t col = jr & 63;
#pragma unroll
        for (uint32_t n = 0; n < 32; ++n) {
          if (n >= Bp) break;
          // token columns >= B (padding) stay 0; the combine weight is
          // applied per column in the down epilogue
          float h = 0.f;
          if (n < B) h = (g[n] / (1.f + __expf(-g[n]))) * up[n];
          const uint16_t hi = f32_to_bf16_rne(h);
          const uint16_t lo = f32_to_bf16_rne(h - bf2f(hi));
          *reinterpret_cast<uint16_t*>(hb + sw128_off(n, col)) = hi;
          *reinterpret_cast<uint16_t*>(hb + sw128_off(Bp + n, col)) = lo;
        }
        fence_proxy_async_global();
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (et == 0) {
          __threadfence();
          atomicAdd(&a.ctr[r.item], 1u);
          mbar_arrive(&rempty_bar[j]);
          if (a.tl) atomicMax(reinterpret_cast<unsigned long long*>(a.tl + 9), (unsigned long long)globaltimer_ns());
        }
      } else {
        float vh[32], vl[32];  // hi / lo columns of every token
#pragma unroll
        for (uint32_t cc = 0; cc < 4; ++cc)
          if (cc * 8 < Bp) {
            um_ld8(ta + cc * 8, vh + cc * 8);
            um_ld8(ta + Bp + cc * 8, vl + cc * 8);
          }
        um_ld_wait();
        um_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[b]);
        const uint32_t row = r.idx * 128 + q * 32 + lane;
        float* pp = ua.part + (size_t)(s_pb[r.item] + r.split) * B * d + row;
#pragma unroll
        for (uint32_t n = 0; n < 32; ++n) {
          if (n >= B) break;
          st_keep(pp + (size_t)n * d, s_wv[r.item * B + n] * (vh[n] + vl[n]), pol_part);
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (et == 0) mbar_arrive(&rempty_bar[j]);
      }
    }
    // this CTA's units are complete
    asm volatile("bar.sync 2, 128;" ::: "memory");
    if (et == 0) {
      __threadfence();
      atomicAdd(&a.ctr[kUmDoneCtr], 1u);
      if (a.tl) {  // first and last CTA done with their units
        const unsigned long long now = globaltimer_ns();
        atomicCAS(reinterpret_cast<unsigned long long*>(a.tl + 14), 0ull, now);
        atomicMax(reinterpret_cast<unsigned long long*>(a.tl + 13), now);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    wait_ctr_ge(&a.ctr[kUmDoneCtr], G, 9u);
    if (a.tl && c == 0) a.tl[11] = globaltimer_ns();
  }
  __syncthreads();
  // epilogue: y[tok][row] = sum over the items in plan order, residual
  {
    // CTA c owns a contiguous range of the flattened [B][d] outputs: every
    // warp load is one 128 B line of a partial
    uint32_t lo, hi;
    share(B * d, c, G, lo, hi);
    const uint32_t np = s_pb[s_ni];
    // the partial forward (items [0, n_local): shared expert + resident hits)
    // is a prefix of the partials in plan order
    const uint32_t np_loc = a.x_pred ? s_pb[min(a.plan->n_local, s_ni)] : 0u;
    for (uint32_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      const uint32_t t = i / d, o = i % d;
      const float* pp = ua.part + (size_t)t * d + o;
      const float xin = bf2f(a.x_in[(size_t)t * d + o]);  // issued before the partials
      // partials in plan order, 32 loads in flight (branch-free: indices past
      // the end reload the last partial and are not added)
      float y = 0.f, y_loc = 0.f;
      for (uint32_t it = 0; it < np; it += 32) {
        float v[32];
#pragma unroll
        for (uint32_t q2 = 0; q2 < 32; ++q2) v[q2] = __ldcg(pp + (size_t)min(it + q2, np - 1) * B * d);
#pragma unroll
        for (uint32_t q2 = 0; q2 < 32; ++q2) {
          if (it + q2 == np_loc) y_loc = y;
          if (it + q2 < np) y += v[q2];
        }
      }
      if (np_loc >= np) y_loc = y;
      const float xo = xin + y;
      a.x_out[(size_t)t * d + o] = f32_to_bf16_rne(xo);
      a.y_out[(size_t)t * d + o] = y;
      if (a.x_pred) a.x_pred[(size_t)t * d + o] = f32_to_bf16_rne(xin + y_loc);
    }
  }
  if (a.tl && c == 0 && threadIdx.x == 0) a.tl[8] = globaltimer_ns();  // CTA 0's final sum done
  if (warp == 1) {
    um_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kUmTmemCols));
  }
  // deferred admissions: staging -> slot once every CTA finished reading
  const uint32_t n_d2d = a.plan->n_d2d;
  if (n_d2d) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&a.ctr[kFfnD2dCtr], 1u);
      wait_ctr_ge(&a.ctr[kFfnD2dCtr], G, 3u);
    }
    __syncthreads();
    const Plan* gp = a.plan;
    const uint64_t nv = gp->d2d_elems / 8;
    for (uint32_t j = 0; j < n_d2d; ++j) {
      const uint4* src = reinterpret_cast<const uint4*>(gp->d2d[j].src);
      uint4* dst = reinterpret_cast<uint4*>(gp->d2d[j].dst);
      for (uint64_t v = c * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)G * blockDim.x)
        dst[v] = ldg_cg(src + v);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (n_d2d) __threadfence();
    const uint32_t prev = atomicAdd(&a.ctr[kFfnExitCtr], 1u);
    if (prev == G - 1) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ffn_done), "r"(a.plan->seq) : "memory");
      if (a.tl) a.tl[2] = globaltimer_ns();
    }
  }
}

// Shared-memory ring for a batch: stages of 32 KB of weights + the largest
// B operand (down: two K-blocks of 2 Bp rows). Returns stages == 0 when the
// shapes do not fit.
struct UmLaunch {
  uint32_t Nx, Bp, stages, stage_bytes, KS, dn_st;
  size_t smem;
};
inline UmLaunch umma_launch_config(uint32_t B, uint32_t d, uint32_t max_items) {
  UmLaunch L{};
  // ~16 x 32 KB stages per gate_up unit, <= 4 per down unit: enough units to
  // spread a few experts over every SM with a short tail
  const uint32_t nkb = d / 64;
  L.KS = 1;
  while (L.KS < 8 && nkb % (2 * L.KS) == 0 && nkb / (2 * L.KS) >= 16) L.KS *= 2;
  // B > 16: more distinct experts (enough units) and twice the split-partial
  // traffic: no K-split (B200, DSV2-Lite all-resident layer period, B = 32:
  // KS 1 / 2 / 4 = 128 / 131 / 135 us; B = 8: 70 / 69 / 74 us)
  if (B > 16) L.KS = 1;
  L.dn_st = 4;
  if (const char* e = getenv("MOEB_UMMA_KS")) {  // tuning knobs
    const uint32_t ks = (uint32_t)atoi(e);
    if (ks >= 1 && nkb % ks == 0) L.KS = ks;
  }
  if (const char* e = getenv("MOEB_UMMA_DNST")) L.dn_st = std::max(1, atoi(e));
  L.Nx = B <= 16 ? 16u : 32u;
  L.Bp = (B + 7) / 8 * 8;
  const uint32_t bmax = std::max(L.Nx * 128, 2 * (2 * L.Bp) * 128);
  L.stage_bytes = (kUmA + bmax + 1023) / 1024 * 1024;
  const size_t wv = (size_t)max_items * B * 4;  // per-item token combine weights
  const size_t budget = 224 * 1024 - 1024 - wv;  // + 1 KB alignment slack
  L.stages = (uint32_t)std::min<size_t>(kUmMaxStages, budget / L.stage_bytes);
  L.smem = (size_t)L.stages * L.stage_bytes + 1024 + wv;
  if (B < 2 || B > 32) L.stages = 0;
  return L;
}

}  // namespace moeb
