// ffn_splitk.cuh — batch-1 grouped SwiGLU FFN without a gate_up -> down
// barrier (sm_100a).
//
// The 2-phase kernel (ffn_tma.cuh) needs every h of an item before any of
// its down rows (a grid barrier, then h staged into every CTA). At batch 1
// this kernel instead splits the down projection over the intermediate
// dimension: the stack stores each expert row-interleaved ([F][3][d]: gate
// row r, up row r, down column r contiguous), and a work unit is ONE
// intermediate row r of an item (3 x 2d bytes: one bulk copy, one ring stage). The consumer warp that
// gets the stage computes h_r = silu(g_r . u) * (u_r . u) on the tensor cores
// (diagonal mma.sync mapping, ffn_tma.cuh) and immediately adds
// (wt * h_r) * Wd^T[r][:] into its own fp32 partial y (registers, d/32 per
// lane). Units are handed out grid-dynamically, so there is no barrier until
// the end: the CTA folds its warps' partials (fixed order), writes them, and
// after one grid barrier each CTA sums its slice of the d outputs over the
// CTAs in fixed order (deterministic) and applies the residual.
//
// With the speculative plan (stack.cu: publish_spec) the units of the
// certain items stream while the decision runs; the final plan's other items
// and the uploaded experts follow on the same ring without any barrier.
#pragma once

#include "ffn_tma.cuh"

namespace moeb {

constexpr int kSkConsumers = 8;
constexpr int kSkThreads = 32 * (1 + kSkConsumers);
constexpr int kSkMaxStages = 24;
constexpr int kSkStages = 16;        // a multiple of the consumer warps (2 stages each); 192 KB at d = 2048
constexpr int kSkMaxYChunks = 8;     // d <= 2048: 8 columns x 8 chunks per lane
constexpr uint32_t kSkStaticUnitRows = 4;  // rows per unit when dealt round-robin (default)
constexpr uint32_t kSkWtShared = 0xffffffffu;  // stage header: combine weight = s_wt_shared (a NaN pattern)
constexpr uint32_t kSkUnitRows = 16;  // rows per grab in the first tier (same-address atomics serialise: keep grabs few)

// silu(g.u) * (u_r.u) for one gate/up row pair in shared memory; every lane
// returns the value
__device__ __forceinline__ float sk_h(const uint16_t* gs, const uint16_t* us_row,
                                      const uint32_t (&xb)[kXrBlocks][2], uint32_t d) {
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  float acc2[4] = {0.f, 0.f, 0.f, 0.f};
  const uint32_t base = diag_addr(smem_u32(gs), smem_u32(us_row));
  const uint32_t nb = d / 128;
#pragma unroll
  for (int b = 0; b < 16; b += 2) {  // d <= 2048
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
  return __fdiv_rn(gu.x, 1.0f + expf(-gu.x)) * gu.y;
}

// the same with the activation's B fragments read from shared memory
__device__ __forceinline__ float sk_h_smem(const uint16_t* gs, const uint16_t* us_row, const uint32_t* su,
                                           uint32_t d) {
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  float acc2[4] = {0.f, 0.f, 0.f, 0.f};
  const int lane = lane_id();
  const uint32_t base = diag_addr(smem_u32(gs), smem_u32(us_row));
  const uint32_t nb = d / 128;
#pragma unroll
  for (int b = 0; b < 16; b += 2) {  // d <= 2048
    if ((uint32_t)b < nb) {
      uint32_t a[4];
      ldsm_x4(base + b * 256, a);
      mma16816(acc, a, su[b * 64 + lane], su[b * 64 + 32 + lane]);
    }
    if ((uint32_t)b + 1 < nb) {
      uint32_t a[4];
      ldsm_x4(base + (b + 1) * 256, a);
      mma16816(acc2, a, su[(b + 1) * 64 + lane], su[(b + 1) * 64 + 32 + lane]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] += acc2[q];
  const float2 gu = diag_reduce(acc);
  return __fdiv_rn(gu.x, 1.0f + expf(-gu.x)) * gu.y;
}

// NC consumer warps; XREG: the activation's B fragments live in registers
// (else in shared memory, which leaves the registers for more warps)
template <int NC, bool XREG>
__global__ void __launch_bounds__(32 * (NC + 1), 1) ffn_splitk_kernel(FfnTArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kSkMaxStages], empty_bar[kSkMaxStages];
  // stage header written by the producer lane before the stage's copy:
  // {item << 16 | 1, row, combine weight} or {0, 0} = end, {0, 1} = snapshot
  __shared__ uint32_t s_hdr[kSkMaxStages][3];
  __shared__ uint32_t s_pre[kMaxItems + 1];  // row prefix of a phase's items
  __shared__ uint32_t s_u[1024];             // the activation (bf16 pairs), d <= 2048
  // partial forward for the next layer's predictor (x_pred): the consumer
  // warps' partials at the snapshot marker, summed in warp order
  __shared__ float s_yloc[2048];
  __shared__ volatile uint32_t s_turn;
  __shared__ uint32_t s_snap;
  // shared-expert rows prefetched before the gate has run: consumers wait
  // for s_uready (u written, shared expert released) and take the combine
  // weight of stages marked kSkWtShared from s_wt_shared
  __shared__ volatile uint32_t s_uready;
  __shared__ float s_wt_shared;
  asm volatile("griddepcontrol.launch_dependents;");
  if (a.tl && blockIdx.x == 0 && threadIdx.x == 0) a.tl[7] = globaltimer_ns();
  const uint32_t G = gridDim.x, c = blockIdx.x;
  // MOEB_FFN_TSTAMP: per-CTA phase stamps [G][8] of the launch (diagnostics)
  uint64_t* const ts = a.tstamp ? a.tstamp + (size_t)c * 8 : nullptr;
  if (ts && threadIdx.x == 0) ts[0] = globaltimer_ns();
  const uint32_t d = a.d, S = a.stages, SB = a.stage_bytes;
  const int warp = warp_id(), lane = lane_id();
  unsigned char* ring = smem_raw;
  Plan* p = reinterpret_cast<Plan*>(smem_raw + S * SB);
  uint32_t dlo, dhi;
  share(d, c, G, dlo, dhi);
  if (threadIdx.x == 0) {
    s_turn = 0;
    s_snap = 0;
    s_uready = 0;
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // residual inputs of this CTA's outputs (written by the previous FFN)
  float xin_pre = 0.f;
  if (threadIdx.x < dhi - dlo) xin_pre = bf2f(a.x_in[dlo + threadIdx.x]);
  const bool spec = a.spec_plan != nullptr;
  if (!spec) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t* src = reinterpret_cast<const uint64_t*>(a.plan);
    uint64_t* dst = reinterpret_cast<uint64_t*>(p);
    for (uint32_t i = threadIdx.x; i < a.plan_smem / 8; i += blockDim.x) dst[i] = src[i];
    if (a.tl && c == 0 && threadIdx.x == 0) a.tl[0] = globaltimer_ns();
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // warp 0: lane 0 streams, all lanes help fetching plans
    const uint64_t pol = l2_evict_first_policy();
    uint32_t k = 0;
    auto acquire = [&]() -> uint32_t {
      const uint32_t st = k % S;
      mbar_wait(&empty_bar[st], ((k / S) & 1) ^ 1);
      return st;
    };
    auto issue_row = [&](uint32_t ii, uint32_t r) {  // lane 0
      const Item& it = p->items[ii];
      const uint32_t F = it.F;
      const uint32_t st = acquire();
      s_hdr[st][0] = (ii << 16) | 1u;
      s_hdr[st][1] = r;
      s_hdr[st][2] = __float_as_uint(it.wt[0]);  // consumers never read the plan (the producer rewrites it)
      unsigned char* dst = ring + st * SB;
      (void)F;
      // row-interleaved layout: [gate r | up r | down column r] contiguous
      mbar_expect_tx(&full_bar[st], 3 * d * 2);
      bulk_g2s(dst, it.w + (size_t)r * 3 * d, 3 * d * 2, &full_bar[st], pol);
      ++k;
    };
    // units of items [i0, i1) handed out by grid counter ctr[ci]
    auto stream = [&](uint32_t i0, uint32_t i1, uint32_t ci, bool small_units) {
      if (lane == 0) {
        uint32_t rows = 0;
        for (uint32_t i = i0; i < i1; ++i) {
          s_pre[i] = rows;
          rows += p->items[i].F;
        }
        s_pre[i1] = rows;
        // guided self-scheduling in three tiers: big units (few same-address
        // atomics, which serialise in L2) for the first 70% of the rows,
        // 8-row units for the next 25%, 2-row units for the tail, so every SM
        // runs out of work within about a microsecond of the others
        // (an uploaded expert alone — ~10 rows per SM — goes out in 2-row
        // units: its completion is on the critical path after the upload)
        const bool det = a.deterministic != 0;
        if (det && !a.unit_rows) {
          // static mode (default): CTA c streams the contiguous rows
          // [rows c / G, rows (c + 1) / G) of this phase — equal shares, every
          // CTA on one long run of DRAM pages (measured faster than dealing
          // 4-row units round-robin: 4 / 8 / 16-row units 35.2 / 34.1 / 33.4 us
          // per all-resident layer, finer units slower), and a fixed row ->
          // (CTA, ring step) map: bitwise-reproducible partial sums
          const uint32_t r0 = (uint32_t)((uint64_t)rows * c / G), r1 = (uint32_t)((uint64_t)rows * (c + 1) / G);
          uint32_t ii = i0;
          for (uint32_t row = r0; row < r1; ++row) {
            while (s_pre[ii + 1] <= row) ++ii;
            issue_row(ii, row - s_pre[ii]);
          }
        } else {
          const uint32_t ub = a.unit_rows ? a.unit_rows : (det ? kSkStaticUnitRows : kSkUnitRows);
          const uint32_t n1 = small_units ? 0 : det ? rows / ub : (rows * 70 / 100) / ub, e1 = n1 * ub;
          const uint32_t n2 = small_units || det ? 0 : (rows * 95 / 100 > e1 ? rows * 95 / 100 - e1 : 0) / 8, e2 = e1 + n2 * 8;
          const uint32_t n_units = n1 + n2 + (rows - e2 + 1) / 2;
          uint32_t* ctr = a.ctr + ci;
          // MOEB_SK_UNIT=n (static): unit u of n rows belongs to CTA u % G;
          // MOEB_DYNAMIC_ROWS=1: units grabbed from a grid counter
          uint32_t u0 = det ? c : atomicAdd(ctr, 1u), u1 = det ? c + G : atomicAdd(ctr, 1u);
          uint32_t ii = i0;
          while (u0 < n_units) {
            const uint32_t cur = u0;
            u0 = u1;
            u1 = det ? u1 + G : atomicAdd(ctr, 1u);
            uint32_t r0, r1;
            if (cur < n1) { r0 = cur * ub; r1 = r0 + ub; }
            else if (cur < n1 + n2) { r0 = e1 + (cur - n1) * 8; r1 = r0 + 8; }
            else { r0 = e2 + (cur - n1 - n2) * 2; r1 = min(rows, r0 + 2); }
            for (uint32_t row = r0; row < r1; ++row) {
              while (s_pre[ii + 1] <= row) ++ii;
              issue_row(ii, row - s_pre[ii]);
            }
          }
        }
      }
      __syncwarp();
    };
    auto fetch = [&](const Plan* gp, uint32_t from, uint32_t words) {  // all lanes of warp 0
      const uint64_t* src = reinterpret_cast<const uint64_t*>(gp);
      uint64_t* dst = reinterpret_cast<uint64_t*>(p);
      for (uint32_t i = from + lane; i < words; i += 32) dst[i] = __ldcg(src + i);
      __syncwarp();
    };
    auto wait_flag = [&](const uint32_t* f, uint32_t slot) {
      if (lane == 0) {
        const uint64_t t0 = globaltimer_ns();
        while (ld_acquire_u32(f) != a.seq) {
          __nanosleep(32);
          if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 5u); break; }
        }
        if (a.tl && c == 0) a.tl[slot] = globaltimer_ns();
      }
      __syncwarp();
    };
    auto load_u = [&]() {  // all lanes of warp 0; u is valid once a plan is
      if (!XREG)
        for (uint32_t i = lane; i < d / 2; i += 32) s_u[i] = __ldcg(reinterpret_cast<const uint32_t*>(a.u) + i);
      __syncwarp();
    };
    uint32_t n_spec = 0;
    if (!spec) load_u();
    if (spec) {
      const uint32_t hdr = (uint32_t)(offsetof(Plan, items) / 8), iw = (uint32_t)(sizeof(Item) / 8);
      uint32_t n0 = 0;
      if (a.shared_first && XREG && a.shared_w && a.deterministic && !a.unit_rows) {
        // the shared expert's weights do not depend on the gate: this CTA's
        // first ring-full of its rows is issued at once (HBM is idle while
        // the gate and the classification run), the rest after the release
        // (same rows, same ring steps as stream(): bitwise-identical sums)
        const uint32_t rows = a.shared_F;
        const uint32_t r0 = (uint32_t)((uint64_t)rows * c / G), r1 = (uint32_t)((uint64_t)rows * (c + 1) / G);
        const uint32_t pre = min(r1 - r0, S);
        if (lane == 0) {
          Item& it0 = p->items[0];
          it0.w = a.shared_w;
          it0.F = rows;
          it0.wt[0] = __uint_as_float(kSkWtShared);
          for (uint32_t r = r0; r < r0 + pre; ++r) issue_row(0, r);
        }
        __syncwarp();
        wait_flag(a.spec_flag + 2, 6);
        fetch(a.spec_plan, hdr, hdr + iw);
        if (lane == 0) {
          s_wt_shared = p->items[0].wt[0];
          __threadfence_block();
          s_uready = 1;
          for (uint32_t r = r0 + pre; r < r1; ++r) issue_row(0, r);
        }
        __syncwarp();
        if (ts && lane == 0) ts[1] = globaltimer_ns();
        n0 = 1;
        wait_flag(a.spec_flag, 9);
        if (ts && lane == 0) ts[2] = globaltimer_ns();
      } else if (a.shared_first) {
        // the shared expert, released right after the gate
        wait_flag(a.spec_flag + 2, 6);
        if (lane == 0) s_uready = 1;
        load_u();
        fetch(a.spec_plan, hdr, hdr + iw);
        stream(0, 1, kFfnSpecGuCtr, false);
        if (ts && lane == 0) ts[1] = globaltimer_ns();
        n0 = 1;
        wait_flag(a.spec_flag, 9);
        if (ts && lane == 0) ts[2] = globaltimer_ns();
      } else {
        wait_flag(a.spec_flag, 6);
        load_u();
      }
      // the certain items while the decision runs
      n_spec = ld_acquire_u32(&a.spec_plan->n_spec);
      fetch(a.spec_plan, hdr + n0 * iw, hdr + n_spec * iw);
      stream(n0, n_spec, kFfnSpecGuCtr, false);
      if (ts && lane == 0) ts[3] = globaltimer_ns();
      // the final plan: its first n_spec items are the speculative ones
      wait_flag(a.spec_flag + 1, 0);
      if (ts && lane == 0) ts[4] = globaltimer_ns();
      const uint32_t hdr_words = (uint32_t)(offsetof(Plan, items) / 8);
      fetch(a.plan, 0, hdr_words);
      fetch(a.plan, hdr_words + n_spec * (uint32_t)(sizeof(Item) / 8), a.plan_smem / 8);
    }
    const uint32_t n_items = p->n_items, n_ready = p->n_ready;
    stream(n_spec, n_ready, kFfnGuCtr, false);
    // snapshot marker (one per consumer warp) right before the first item
    // that is not the shared expert or a resident hit: the partial forward
    auto snapshot = [&]() {
      if (lane == 0) {
        for (int w = 0; w < NC; ++w) {
          const uint32_t st = acquire();
          s_hdr[st][0] = 0;
          s_hdr[st][1] = 1;
          mbar_arrive(&full_bar[st]);
          ++k;
        }
        s_snap = 1;
      }
      __syncwarp();
    };
    const uint32_t n_local = a.x_pred ? p->n_local : n_items;
    // the uploaded experts, as they land; units from the item's own counter
    for (uint32_t ii = n_ready; ii < n_items; ++ii) {
      if (ii == n_local) snapshot();
      if (lane == 0 && p->items[ii].spec) {  // a speculative upload buffer
        const uint32_t sp = p->items[ii].spec, b = sp >> 31, g = sp & 0x7fffffffu;
        const uint64_t t0 = globaltimer_ns();
        while ((int32_t)(ld_acquire_u32(a.spec_done + b) - g) < 0) {
          __nanosleep(128);
          if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 8u); break; }
        }
        if (a.tl && c == 0) a.tl[1] = globaltimer_ns();
        asm volatile("fence.proxy.async;" ::: "memory");
      }
      if (lane == 0 && p->items[ii].wait) {
        const uint64_t t0 = globaltimer_ns();
        while ((int32_t)(ld_acquire_u32(a.copies_done) - p->items[ii].wait) < 0) {
          __nanosleep(128);
          if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 1u); break; }
        }
        if (a.tl && c == 0) a.tl[1] = globaltimer_ns();
        // the uploaded bytes are read by the async (bulk-copy) proxy next
        asm volatile("fence.proxy.async;" ::: "memory");
      }
      __syncwarp();
      stream(ii, ii + 1, ii, true);
    }
    if (ts && lane == 0) ts[5] = globaltimer_ns();
    if (lane == 0) {
      for (int w = 0; w < NC; ++w) {  // one end marker per consumer warp
        const uint32_t st = acquire();
        s_hdr[st][0] = 0;
        s_hdr[st][1] = 0;
        mbar_arrive(&full_bar[st]);
        ++k;
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    // ring step k belongs to warp k % NC
    const uint32_t cw = warp - 1, ych = d / 256;
    float y[kSkMaxYChunks][8];
#pragma unroll
    for (int j = 0; j < kSkMaxYChunks; ++j)
#pragma unroll
      for (int q = 0; q < 8; ++q) y[j][q] = 0.f;
    uint32_t xb[XREG ? kXrBlocks : 1][2];
    bool have_x = false;
    uint32_t k_det = cw;
    for (;;) {
      // step k belongs to warp k % NC and the stage count is a multiple of
      // NC: a slot always has the same warp, which consumes its phases in
      // order, so a parity wait can never match a stale phase (a dynamic
      // claim could, if an older copy into that slot completed late)
      const uint32_t k = k_det;
      k_det += NC;
      const uint32_t st = k % S;
      mbar_wait(&full_bar[st], (k / S) & 1);
      const uint32_t h0 = s_hdr[st][0];
      if (h0 == 0) {
        if (s_hdr[st][1] == 1) {
          // snapshot: add this warp's partial into s_yloc, warps in order
          while (s_turn != cw) {}
#pragma unroll
          for (int j = 0; j < kSkMaxYChunks; ++j)
            if ((uint32_t)j < ych)
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                float& dst = s_yloc[j * 256 + lane * 8 + q];
                dst = cw == 0 ? y[j][q] : dst + y[j][q];
              }
          __syncwarp();
          __threadfence_block();
          if (lane == 0) {
            s_turn = cw + 1;
            mbar_arrive(&empty_bar[st]);
          }
          continue;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
        break;
      }
      if (XREG && !have_x) {  // u: the gate phase wrote it before either plan was released
        if (a.shared_first) {  // (rows may have been issued before the release)
          const uint64_t t0 = globaltimer_ns();
          while (!s_uready) {
            __nanosleep(20);
            if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 9u); break; }
          }
          __threadfence_block();
        }
        const uint32_t* u32w = reinterpret_cast<const uint32_t*>(a.u);
#pragma unroll
        for (int b = 0; b < (XREG ? kXrBlocks : 1); ++b) {
          const bool in = (uint32_t)b < d / 128;
          xb[b][0] = in ? __ldcg(u32w + b * 64 + lane) : 0u;
          xb[b][1] = in ? __ldcg(u32w + b * 64 + 32 + lane) : 0u;
        }
        have_x = true;
      }
      const float wt = s_hdr[st][2] == kSkWtShared ? s_wt_shared : __uint_as_float(s_hdr[st][2]);
      const uint16_t* base = reinterpret_cast<const uint16_t*>(ring + st * SB);
      if constexpr (XREG) {
        if (!(a.dbg & 1)) {
          // the down column to registers and the gate/up MMAs, then the
          // stage goes back to the producer (the arrive's release orders
          // the reads) before the reduction, silu and the down FMAs
          const uint4* wd = reinterpret_cast<const uint4*>(base + 2 * d);
          uint4 wdr[kSkMaxYChunks];
#pragma unroll
          for (int j = 0; j < kSkMaxYChunks; ++j)
            if ((uint32_t)j < ych) wdr[j] = wd[j * 32 + lane];
          float acc[4] = {0.f, 0.f, 0.f, 0.f}, acc2[4] = {0.f, 0.f, 0.f, 0.f};
          const uint32_t dbase = diag_addr(smem_u32(base), smem_u32(base + d));
          const uint32_t nb = d / 128;
#pragma unroll
          for (int b = 0; b < 16; b += 2) {
            if ((uint32_t)b < nb) {
              uint32_t f[4];
              ldsm_x4(dbase + b * 256, f);
              mma16816(acc, f, xb[b][0], xb[b][1]);
            }
            if ((uint32_t)b + 1 < nb) {
              uint32_t f[4];
              ldsm_x4(dbase + (b + 1) * 256, f);
              mma16816(acc2, f, xb[b + 1][0], xb[b + 1][1]);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[st]);
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] += acc2[q];
          const float2 gu = diag_reduce(acc);
          const float s = wt * (__fdiv_rn(gu.x, 1.0f + expf(-gu.x)) * gu.y);
#pragma unroll
          for (int j = 0; j < kSkMaxYChunks; ++j) {
            if ((uint32_t)j < ych) {
              const uint4 w = wdr[j];
              y[j][0] = fmaf(s, __uint_as_float(w.x << 16), y[j][0]);
              y[j][1] = fmaf(s, __uint_as_float(w.x & 0xffff0000u), y[j][1]);
              y[j][2] = fmaf(s, __uint_as_float(w.y << 16), y[j][2]);
              y[j][3] = fmaf(s, __uint_as_float(w.y & 0xffff0000u), y[j][3]);
              y[j][4] = fmaf(s, __uint_as_float(w.z << 16), y[j][4]);
              y[j][5] = fmaf(s, __uint_as_float(w.z & 0xffff0000u), y[j][5]);
              y[j][6] = fmaf(s, __uint_as_float(w.w << 16), y[j][6]);
              y[j][7] = fmaf(s, __uint_as_float(w.w & 0xffff0000u), y[j][7]);
            }
          }
          continue;
        }
      }
      if (!(a.dbg & 1)) {
        float hv;
        if constexpr (XREG) hv = sk_h(base, base + d, xb, d);
        else hv = sk_h_smem(base, base + d, s_u, d);
        const float s = wt * hv;
        const uint4* wd = reinterpret_cast<const uint4*>(base + 2 * d);
#pragma unroll
        for (int j = 0; j < kSkMaxYChunks; ++j) {
          if ((uint32_t)j < ych) {
            const uint4 w = wd[j * 32 + lane];
            y[j][0] = fmaf(s, __uint_as_float(w.x << 16), y[j][0]);
            y[j][1] = fmaf(s, __uint_as_float(w.x & 0xffff0000u), y[j][1]);
            y[j][2] = fmaf(s, __uint_as_float(w.y << 16), y[j][2]);
            y[j][3] = fmaf(s, __uint_as_float(w.y & 0xffff0000u), y[j][3]);
            y[j][4] = fmaf(s, __uint_as_float(w.z << 16), y[j][4]);
            y[j][5] = fmaf(s, __uint_as_float(w.z & 0xffff0000u), y[j][5]);
            y[j][6] = fmaf(s, __uint_as_float(w.w << 16), y[j][6]);
            y[j][7] = fmaf(s, __uint_as_float(w.w & 0xffff0000u), y[j][7]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[st]);
    }
    // every stage of this warp is consumed: park the partial in the ring
    // after the whole CTA is done with it
    asm volatile("bar.sync 1, %0;" ::"n"(NC * 32) : "memory");
    float* scratch = reinterpret_cast<float*>(ring) + (size_t)cw * d;
#pragma unroll
    for (int j = 0; j < kSkMaxYChunks; ++j)
      if ((uint32_t)j < ych) {
        float4* o = reinterpret_cast<float4*>(scratch + j * 256 + lane * 8);
        o[0] = make_float4(y[j][0], y[j][1], y[j][2], y[j][3]);
        o[1] = make_float4(y[j][4], y[j][5], y[j][6], y[j][7]);
      }
  }
  __syncthreads();
  if (ts && threadIdx.x == 0) ts[6] = globaltimer_ns();
  if (a.tl && c == 0 && threadIdx.x == 0) a.tl[11] = globaltimer_ns();
  if (a.tl && threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(&a.tl[13]), (unsigned long long)globaltimer_ns());
  // this CTA's partial y (warps summed in order) -> global partials [G][d]
  float* part = a.h;
  float* part_loc = a.h + (size_t)G * d;  // partial-forward partials (x_pred)
  const bool snap = s_snap != 0;
  {
    const float* scratch = reinterpret_cast<const float*>(ring);
    for (uint32_t o = threadIdx.x; o < d; o += blockDim.x) {
      float s = scratch[o];
#pragma unroll
      for (int w = 1; w < NC; ++w) s += scratch[(size_t)w * d + o];
      part[(size_t)c * d + o] = s;
      if (snap) part_loc[(size_t)c * d + o] = s_yloc[o];
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&a.ctr[kFfnRedCtr], 1u);
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_u32(&a.ctr[kFfnRedCtr]) < G) {
      __nanosleep(20);
      if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 2u); break; }
    }
    if (a.tl && c == 0) a.tl[14] = globaltimer_ns();
    // every CTA has finished reading expert slots (it passed its consumer
    // loop before arriving): without deferred copies, ffn_done can be
    // released now instead of after a second exit barrier
    if (c == 0 && p->n_d2d == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ffn_done), "r"(p->seq) : "memory");
    }
  }
  __syncthreads();
  // outputs [dlo, dhi): sum of the CTA partials, residual. The [G][no]
  // block this CTA needs is gathered with coalesced loads (consecutive
  // threads read consecutive outputs of one partial, all loads in flight
  // together) into shared memory; then each output thread sums its G values
  // in 8 interleaved chains combined in a fixed order (deterministic).
  {
    const uint32_t no = dhi - dlo;  // <= 16 (d <= 2048, G >= 128)
    float* gath = reinterpret_cast<float*>(ring);  // [G][16]
    auto final_sum = [&](const float* src) -> float {
      // item t = (partial t / 16, output t % 16): half-warps read one
      // partial's outputs, every load in flight at once
      constexpr uint32_t kIn = 9;
      const uint32_t n = G * 16;
      for (uint32_t t0 = threadIdx.x; t0 < n; t0 += kIn * blockDim.x) {
        float v[kIn];
#pragma unroll
        for (uint32_t q = 0; q < kIn; ++q) {
          const uint32_t t = t0 + q * blockDim.x, cc = t >> 4, o = t & 15u;
          v[q] = (t < n && o < no) ? __ldcg(src + (size_t)cc * d + dlo + o) : 0.f;
        }
#pragma unroll
        for (uint32_t q = 0; q < kIn; ++q) {
          const uint32_t t = t0 + q * blockDim.x;
          if (t < n) gath[t] = v[q];
        }
      }
      __syncthreads();
      float yv = 0.f;
      if (threadIdx.x < no) {
        // 8 interleaved chains in a fixed order (deterministic)
        float ch[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        uint32_t cc = 0;
        for (; cc + 8 <= G; cc += 8)
#pragma unroll
          for (uint32_t q = 0; q < 8; ++q) ch[q] += gath[(cc + q) * 16 + threadIdx.x];
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q)
          if (cc + q < G) ch[q] += gath[(cc + q) * 16 + threadIdx.x];
        yv = ((ch[0] + ch[1]) + (ch[2] + ch[3])) + ((ch[4] + ch[5]) + (ch[6] + ch[7]));
      }
      __syncthreads();
      return yv;
    };
    const float yv = final_sum(part);
    if (threadIdx.x < no) {
      const uint32_t o = dlo + threadIdx.x;
      a.x_out[o] = f32_to_bf16_rne(xin_pre + yv);
      a.y_out[o] = yv;
      if (a.x_pred && !snap) a.x_pred[o] = f32_to_bf16_rne(xin_pre + yv);  // every item was local
    }
    if (a.x_pred && snap) {  // the partial forward: the same sum over the snapshot partials
      const float yl = final_sum(part_loc);
      if (threadIdx.x < no) a.x_pred[dlo + threadIdx.x] = f32_to_bf16_rne(xin_pre + yl);
    }
  }
  // deferred admissions: staging -> slot (every CTA passed the barrier above,
  // so every read of the staging copies is done)
  const uint32_t n_d2d = p->n_d2d;
  if (n_d2d) {
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
  if (threadIdx.x == 0) {
    if (n_d2d) {
      // the staging -> slot copies must be visible before ffn_done releases
      // the copy stream's prefetches into those slots: last CTA out signals
      __threadfence();
      const uint32_t prev = atomicAdd(&a.ctr[kFfnExitCtr], 1u);
      if (prev == G - 1) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ffn_done), "r"(p->seq) : "memory");
      }
    }
    if (a.tl && c == 0) a.tl[2] = globaltimer_ns();
    if (ts) ts[7] = globaltimer_ns();
  }
}

// Launch shape: the ring (kSkStages stages of 3 rows), the plan copy, and
// the reduction scratch (aliases the ring).
inline FfnLaunch ffn_splitk_config(uint32_t d, uint32_t E, uint32_t top_k, int consumers, bool deterministic) {
  FfnLaunch L{};
  (void)consumers;  // 4-12 consumer warps measured within 0.5 us of each other: 8
  L.fn = ffn_splitk_kernel<8, true>;
  L.threads = 32 * 9;
  L.stage_bytes = 3 * 2 * d;
  // step k -> warp k % NC: the stage count is a multiple of NC
  (void)deterministic;
  const uint32_t nc = L.threads / 32 - 1;
  uint32_t want = kSkStages;
  if (const char* v = getenv("MOEB_SK_STAGES")) want = (uint32_t)atoi(v);  // experiment knob
  L.stages = std::min<uint32_t>(kSkMaxStages, std::max<uint32_t>(nc, want / nc * nc));
  const uint32_t max_items = 1 + std::min(E, top_k);
  L.plan_smem = (uint32_t)((offsetof(Plan, items) + (size_t)max_items * sizeof(Item) + 15) & ~(size_t)15);
  L.x_smem = 0;
  L.acc_rows = 0;
  L.hbuf_bytes = 0;
  const size_t ring = std::max<size_t>((size_t)L.stages * L.stage_bytes, (size_t)(L.threads / 32 - 1) * d * 4);
  L.stage_bytes = (uint32_t)(ring / L.stages);  // the scratch must fit in the ring
  L.smem = ring + L.plan_smem;
  return L;
}

}  // namespace moeb
