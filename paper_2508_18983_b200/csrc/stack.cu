// stack.cu — the MoE decode stack: per layer gate -> decide(+plan) -> FFN on
// the compute stream; expert uploads on a dedicated copy stream issued by a
// host copy thread from a mapped-memory mailbox the decide kernel fills.
//
// Per (iteration, layer) the decide kernel runs the bit-exact decision step
// (decide.cuh) on the fp32 router scores it just computed, turns the outcome
// into (a) an FFN plan (items = shared expert + distinct selected experts with
// token lists and combine weights) and (b) upload commands, and publishes (b)
// in a pinned ring the copy thread polls. Uploads are pinned-host
// cudaMemcpyAsync H2D copies into the cache slot the device chose (or into a
// staging buffer for BA-streamed / deferred / pass-through experts), each
// followed by cuStreamWriteValue32(copies_done = id); the FFN waits item by
// item on that counter. Prefetches for the next layer carry
// cuStreamWaitValue32(ffn_done >= step) so a slot is never overwritten while
// a running FFN may read it.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>  // environ

#include "../../include/moesched_b200.h"
#include "decide.cuh"
#include "engine_host.h"
#include "host_common.h"
#include "layer.cuh"
#include "ffn_tma.cuh"
#include "ffn_splitk.cuh"
#include "ffn_umma.cuh"
#include "prefill.cuh"
#include "weights.cuh"

namespace moeb {

constexpr int kMaxCmds = 3 * kMaxE + 8;
constexpr int8_t kStageSpec = 127;  // stage_of marker: the expert sits in the speculative buffer
constexpr uint32_t kRing = 1024;

// Stream memory operations come from the driver API; resolve them through
// the runtime so libmoeb.so itself does not link libcuda (it must load on
// hosts without a driver, e.g. for the CPU-side ABI checks).
using PFN_write32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PFN_wait32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_write32 p_write32 = nullptr;
static PFN_wait32 p_wait32 = nullptr;

static void load_stream_memops() {
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q1, q2;
    void* f1 = nullptr;
    void* f2 = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f1, cudaEnableDefault, &q1) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess ||
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &f2, cudaEnableDefault, &q2) != cudaSuccess ||
        q2 != cudaDriverEntryPointSuccess) {
      err = "driver entry points cuStreamWriteValue32/cuStreamWaitValue32 unavailable";
      return;
    }
    p_write32 = reinterpret_cast<PFN_write32>(f1);
    p_wait32 = reinterpret_cast<PFN_wait32>(f2);
  });
  if (!p_write32 || !p_wait32) throw Error(5, err);
}

struct MailCmd {
  uint64_t src_off;   // byte offset into the pinned host pool
  uint64_t dst;       // device address
  uint64_t bytes;
  uint32_t id;        // upload id; copies_done := id after the copy
  uint32_t wait_ffn;  // nonzero: copy waits for ffn_done >= wait_ffn
  uint32_t kind;      // 0 upload; 1 speculative upload (the copy thread runs it in chunks
                      // while the copy engine is otherwise idle); 2 promote: a speculative
                      // upload is needed now, issue whatever is left of it
  uint32_t gen, buf;  // speculative: generation, buffer (spec_done[buf] := gen when landed)
  uint32_t pad;
};
// A command on the wire (the mapped host ring): six 64-bit words, each
// carrying the low 16 bits of the entry's sequence in its top 16 bits.
// 64-bit aligned stores arrive whole, so the copy thread takes a command
// once every word shows the entry's tag — no system-scope fence on the
// device's publish path (measured ~1.5-2.5 us per upload layer), and a
// word left over from the entry kRing sequences earlier carries another tag.
struct __align__(16) WireCmd {
  uint64_t w[6];  // src_off | dst | bytes, kind, buf | id | wait_ffn | gen  (payload <= 48 bits each)
};
static_assert(sizeof(WireCmd) == sizeof(MailCmd), "wire command size");
__host__ __device__ inline uint64_t wire_tag(uint64_t mseq) { return (mseq & 0xffffull) << 48; }
__device__ __forceinline__ void put_wire(WireCmd* wc, const MailCmd& c, uint64_t mseq) {
  const uint64_t t = wire_tag(mseq), m = (1ull << 48) - 1;
  const uint64_t w0 = (c.src_off & m) | t, w1 = (c.dst & m) | t;
  const uint64_t w2 = (c.bytes & ((1ull << 40) - 1)) | ((uint64_t)(c.kind & 15u) << 40) | ((uint64_t)(c.buf & 15u) << 44) | t;
  const uint64_t w3 = (uint64_t)c.id | t, w4 = (uint64_t)c.wait_ffn | t, w5 = (uint64_t)c.gen | t;
  // three 16-byte stores to the mapped ring (each 8-byte half arrives whole)
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(wc->w), "l"(w0), "l"(w1) : "memory");
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(wc->w + 2), "l"(w2), "l"(w3) : "memory");
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(wc->w + 4), "l"(w4), "l"(w5) : "memory");
}
// seq word = (sequence << 8) | command count, one 64-bit store
struct MailEntry {
  volatile uint64_t seq;
  uint32_t n, pad;
  WireCmd cmd[kMaxCmds];
};
static_assert(kMaxCmds < 256, "command count is packed in 8 bits");

struct DecideArgs {
  DevCfg cfg;
  EngineState* st;
  LayerState* layers;
  double* hist;
  uint32_t layer;
  const float* logits;        // gate output [B][E+1]
  const float* trace;         // [trace_steps][L][B][E] or null
  uint64_t trace_steps, total_iters;
  int32_t shared_gate, renormalize;
  float routed_scale;
  const uint16_t* shared_w;   // this layer's shared expert or null
  uint32_t S, F, d, slots_alloc;
  uint16_t* slots;            // [L][slots_alloc][expert_elems]
  uint16_t* staging;          // [n_stage][expert_elems]
  uint32_t n_stage;
  uint64_t expert_elems;
  Plan* plan;
  Plan* spec_plan;            // early plan of the certain, ready items (B == 1) or null
  uint32_t* spec_flag;        // := seq once spec_plan is published
  uint32_t* ffn_ctr;
  const uint32_t* copies_done; // upload ids landed so far (written by the copy stream)
  MailEntry* ring;
  const volatile uint64_t* host_ack;
  float* scores_log;          // [rec_cap][B][E] or null
  StepRec* recs;
  TokRec* toks;
  uint64_t rec_cap;
  uint64_t* tl;               // timeline trace record of this layer-step (nullable):
                              // 3 decider entry, 4 uploads published (entry A), 5 end of decide
  uint64_t it;                // decode iteration of this launch (host-tracked)
  uint64_t seq;               // 1-based layer-step sequence number (host-tracked)
  // predictor mode: the prediction of this layer's scores from the previous
  // layer's partial forward (gate CTAs: plogits), logged per step for replay
  uint32_t predictor;
  uint32_t shared_first;      // split-K FFN: the shared expert alone is released right after the gate
  uint32_t spec_up;           // speculative uploads of the next layer's likely miss
  uint16_t* specbuf;          // [2][expert_elems]
  const float* plogits;       // [B][E + 1]
  float* pred_log;            // [rec_cap][B][E] or null
};

struct GateDecideArgs {
  GateArgs g;
  DecideArgs d;
  uint32_t* ticket;           // last-CTA election counter (self-resetting)
};

constexpr int kGdThreads = 256;
constexpr uint32_t kMaxHistSmem = 32 * kMaxE;  // window * E doubles staged in smem

// Shared state of the deciding CTA. Everything the decision step touches
// lives here for the step: engine state, the executing and the prefetch
// target layer (state + score ring), the plan and the upload commands.
struct DecideKSmem {
  DecideSmem d;
  NextSmem n;
  StepScratch s;
  DevCfg cfg;
  EngineState st;
  LayerState ls, tls;
  double hist[kMaxHistSmem], thist[kMaxHistSmem];
  float sc[kMaxB][kMaxE];
  float nsc[kMaxB][kMaxE];
  float sg[kMaxB];
  float denom[kMaxB];
  Plan plan;
  MailCmd cmd[kMaxCmds];
  uint32_t n_cmds;
  uint32_t landed;            // copies_done when the step's state was staged
  volatile uint32_t mail_a;   // mailbox entry A is out (warp 0 -> warp 2)
  uint32_t spec_stage;        // speculative plan: 0 not built, 1 built (release after mailbox A), 2 released
  uint32_t spec_n;            // items in the speculative plan (0: none published)
  uint64_t spec_set;          // routed experts in it
  uint64_t it, seq;
  int last;
  // uploads published early by EarlyPublish (ids + destinations)
  uint32_t load_id[kMaxE], cpu_id[kMaxE];
  uint16_t* load_dst[kMaxE];
  uint16_t* cpu_dst[kMaxE];
  int8_t stage_of[kMaxE];
  uint32_t load_spec[kMaxE], cpu_spec[kMaxE];  // Item::spec of each load / streamed expert
  int32_t spec_slot;          // cache slot the speculative buffer is copied into (-1: none)
  uint32_t spec_buf;
};

__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const volatile uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint16_t* slot_ptr(const DecideArgs& a, uint32_t layer, int slot) {
  return a.slots + ((size_t)layer * a.slots_alloc + (uint32_t)slot) * a.expert_elems;
}

// Copy several global segments into shared memory with every load issued
// before any store (one memory latency for the whole staging phase).
struct StageSeg {
  uint64_t* dst;
  const uint64_t* src;
  uint32_t words;
};
__device__ inline void stage_gather(const StageSeg* segs, int nseg) {
  constexpr int kPer = 20;
  uint32_t total = 0;
  for (int i = 0; i < nseg; ++i) total += segs[i].words;
  for (uint32_t base = 0; base < total; base += kPer * blockDim.x) {
    uint64_t v[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      uint32_t i = base + threadIdx.x + k * blockDim.x;
      if (i < total) {
        int sgi = 0;
        while (i >= segs[sgi].words) { i -= segs[sgi].words; ++sgi; }
        v[k] = segs[sgi].src[i];
      }
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      uint32_t i = base + threadIdx.x + k * blockDim.x;
      if (i < total) {
        int sgi = 0;
        while (i >= segs[sgi].words) { i -= segs[sgi].words; ++sgi; }
        segs[sgi].dst[i] = v[k];
      }
    }
  }
}

template <class T>
__device__ __forceinline__ void cta_copy(T* dst, const T* src) {
  static_assert(sizeof(T) % 8 == 0, "8-byte granular");
  const uint64_t* s = reinterpret_cast<const uint64_t*>(src);
  uint64_t* d = reinterpret_cast<uint64_t*>(dst);
  for (uint32_t i = threadIdx.x; i < sizeof(T) / 8; i += blockDim.x) d[i] = s[i];
}

// The copy thread acknowledges mailbox entries in order; the device only
// re-reads the (PCIe-mapped) acknowledgement when its cached copy is too old.
__device__ __forceinline__ void wait_ring_slot(const DecideArgs& a, uint64_t mseq, uint64_t* ack_cache) {
  if (mseq <= kRing || *ack_cache >= mseq - kRing) return;
  const uint64_t t0 = globaltimer_ns();
  for (;;) {
    *ack_cache = ld_acquire_sys_u64(a.host_ack);
    if (*ack_cache >= mseq - kRing) break;
    __nanosleep(500);
    if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 4u); break; }
  }
}

// Mailbox entry A of a layer-step (sequence 2*seq-1): the demand loads and
// BA-streamed experts, published from inside the decision step the moment
// the lists are final. Entry B (2*seq) carries the prefetches later.
__device__ void publish_spec(const DecideArgs& a, DecideKSmem* sm, const DecideSmem* d, uint64_t mask, bool early);

struct EarlyPublish {
  const DecideArgs* a;
  DecideKSmem* sm;
  __device__ void classified(DecideSmem* d, uint64_t mask) const { publish_spec(*a, sm, d, mask, false); }
  __device__ void classified_early(DecideSmem* d, uint64_t mask) const { publish_spec(*a, sm, d, mask, true); }
  __device__ void plan_ready(DecideSmem* d) const;
  __device__ void prefetched(DecideSmem* d) const;
  __device__ void operator()(DecideSmem* d, uint32_t n_load, uint32_t n_cpu) const {
    if (lane_id() == 0) {
      const DecideArgs& A = *a;
      const uint64_t mseq = 2 * sm->seq - 1;
      MailEntry* me = &A.ring[mseq % kRing];
      wait_ring_slot(A, mseq, &sm->st.ack_cache);
      EngineState* st = &sm->st;
      LayerState* ls = &sm->ls;
      const uint32_t layer = A.layer, E = sm->cfg.E;
      uint32_t si = 0, n = 0;
      for (uint32_t e = 0; e < E; ++e) sm->stage_of[e] = -1;
      sm->spec_slot = -1;
      auto cmd = [&](uint32_t e, uint16_t* dst) {
        const uint32_t id = ++st->next_copy;
        MailCmd c;
        c.src_off = ((uint64_t)layer * E + e) * A.expert_elems * 2;
        c.dst = (uint64_t)dst;
        c.bytes = A.expert_elems * 2;
        c.id = id;
        c.wait_ffn = 0;
        c.kind = 0;
        c.gen = c.buf = c.pad = 0;
        put_wire(&me->cmd[n++], c, mseq);
        return id;
      };
      // the speculative upload meant for this step (buffer seq % 2): an
      // expert this step uploads anyway comes from there instead — the copy
      // thread finishes it at once (promote) and the FFN copies it into its
      // cache slot; decisions are untouched
      const uint32_t sb = (uint32_t)(sm->seq & 1);
      uint32_t sp_e = 0xffffffffu, sp_gen = 0;
      if (A.spec_up && st->sp_valid[sb] && st->sp_layer[sb] == layer && st->sp_it[sb] == sm->it) {
        sp_e = st->sp_expert[sb];
        sp_gen = st->sp_gen[sb];
      }
      st->sp_valid[sb] = 0;
      uint16_t* const sbuf = A.specbuf + (size_t)sb * A.expert_elems;
      auto promote = [&]() {
        MailCmd c;
        c.src_off = c.dst = c.bytes = 0;
        c.id = c.wait_ffn = 0;
        c.kind = 2;
        c.gen = sp_gen;
        c.buf = sb;
        c.pad = 0;
        put_wire(&me->cmd[n++], c, mseq);
        st->sp_hits += 1;
        sp_e = 0xffffffffu;  // one use
      };
      const uint32_t sp_tag = (sb << 31) | sp_gen;
      for (uint32_t i = 0; i < n_load; ++i) {
        const uint32_t e = d->out.load[i];
        const int slot = d->out.load_slot[i];
        if (e == sp_e) {
          promote();
          if (slot >= 0) {
            sm->spec_slot = slot;
            sm->spec_buf = sb;
            ls->slot_copy[slot] = 0;  // filled from the buffer by this step's FFN epilogue
          } else {
            sm->stage_of[e] = kStageSpec;  // a deferred admission copies from the buffer
            sm->spec_buf = sb;
          }
          sm->load_id[i] = 0;
          sm->load_spec[i] = sp_tag;
          sm->load_dst[i] = sbuf;
          continue;
        }
        uint16_t* dst;
        if (slot >= 0) {
          dst = slot_ptr(A, layer, slot);
        } else {
          sm->stage_of[e] = (int8_t)si;
          dst = A.staging + (size_t)(si++ % A.n_stage) * A.expert_elems;
        }
        const uint32_t id = cmd(e, dst);
        if (slot >= 0) ls->slot_copy[slot] = id;
        sm->load_id[i] = id;
        sm->load_spec[i] = 0;
        sm->load_dst[i] = dst;
      }
      for (uint32_t i = 0; i < n_cpu; ++i) {
        if (d->out.cpu[i] == sp_e) {  // BA-streamed: computed straight from the buffer
          promote();
          sm->cpu_id[i] = 0;
          sm->cpu_spec[i] = sp_tag;
          sm->cpu_dst[i] = sbuf;
          continue;
        }
        uint16_t* dst = A.staging + (size_t)(si++ % A.n_stage) * A.expert_elems;
        sm->cpu_id[i] = cmd(d->out.cpu[i], dst);
        sm->cpu_spec[i] = 0;
        sm->cpu_dst[i] = dst;
      }
      me->n = n;
#ifdef MOEB_PROFILE_PHASES
      const uint64_t tf0 = ptimer();
#endif
      // no system fence: the copy thread checks every command word's tag
      me->seq = (mseq << 8) | n;
      if (A.tl) {
        A.tl[4] = globaltimer_ns();
        A.tl[15] = n;  // uploads published by this step
      }
      atomicExch(const_cast<uint32_t*>(&sm->mail_a), 1u);  // warp 2 polls it (publish_spec)
#ifdef MOEB_PROFILE_PHASES
      st->prof[13] += ptimer() - tf0;
#endif
    }
    __syncwarp();
  }
};

// Speculative plan (batch 1): right after classification the shared expert
// and every routed expert certain to be selected — the top-score class with
// substitution on (route pass 1, router.cpp:114-120), the k actives without
// (plain_top_k) — that is resident in the pre-route snapshot with its upload
// landed is final: hits are shielded (pipeline.cpp:196-201), so its slot
// cannot change in this step. Publishing these lets the FFN kernel (already
// resident via PDL) stream them while the rest of the decision runs.
// early: called by the last warp right after classification (beside route
// pass 2, batch < warps); the plan is built and, unless it must wait for the
// step's uploads to be handed off, released there. Otherwise (or if it was
// not called early) warp 2 finishes it after the fork.
__device__ void publish_spec(const DecideArgs& a, DecideKSmem* sm, const DecideSmem* d, uint64_t mask, bool early) {
  if (lane_id() != 0) return;  // one lane of warp 2 (or the last warp), beside the routing on warp 0
  if (!early && sm->spec_stage == 2) return;
  if (!early && sm->spec_stage == 1) {
    const uint64_t t0 = globaltimer_ns();
    while (!atomicAdd(const_cast<uint32_t*>(&sm->mail_a), 0u) && globaltimer_ns() - t0 < kSpinLimitNs) {}
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.spec_flag), "r"((uint32_t)sm->seq) : "memory");
    sm->spec_stage = 2;
    return;
  }
  sm->spec_n = 0;
  sm->spec_set = 0;
  if (!a.spec_plan) return;
  const DevCfg& cfg = sm->cfg;
  const LayerState* ls = &sm->ls;
  // batch: the union over the tokens (an expert no token ends up selecting
  // stays in the final plan with no tokens: zero combine weights)
  uint64_t certain = 0;
  for (uint32_t t = 0; t < cfg.B; ++t) certain |= cfg.er ? d->top[t] : d->act[t];
  // a certain expert that is not resident means uploads this step: the
  // speculative stream would then only compete for HBM with the decision
  // (the FFN cannot finish before the upload lands anyway), so the plan is
  // released once warp 0 has handed the uploads to the copy engine
  const bool uploads = (certain & ~mask) != 0;
  certain &= mask;  // the pre-route snapshot (warp 0 may be admitting meanwhile)
  Plan* sp = a.spec_plan;
  uint32_t n = 0;
  auto item = [&](const uint16_t* w, uint32_t F, uint32_t kind, uint32_t e, float wt) {
    Item& it = sp->items[n++];
    it.w = w;
    it.F = F;
    it.wait = 0;
    it.n_tok = 1;
    it.kind = kind;
    it.expert = e;
    it.tok[0] = 0;
    it.wt[0] = wt;
  };
  if (a.shared_w) {
    if (a.shared_first) ++n;  // item 0 went out right after the gate (release_shared)
    else item(a.shared_w, a.S, 0, 0, a.shared_gate ? sm->sg[0] : 1.0f);
  }
  uint64_t set = 0;
  for (uint64_t m = certain; m; m &= m - 1) {
    const uint32_t e = __ffsll((long long)m) - 1;
    const int slot = ls->slot_of[e];
    const uint32_t w = ls->slot_copy[slot];
    if (w && (int32_t)(sm->landed - w) < 0) continue;  // upload still in flight
    item(slot_ptr(a, a.layer, slot), a.F, 1, e, __fmul_rn(sm->sc[0][e], a.routed_scale));
    set |= 1ull << e;
  }
  sp->n_items = n;
  sp->n_ready = n;
  sp->n_spec = n;
  sp->seq = (uint32_t)sm->seq;
  sm->spec_n = n;
  sm->spec_set = set;
  // (the release store below orders this lane's plan writes)
  if (uploads && early) {
    sm->spec_stage = 1;  // warp 2 releases it once mailbox A is out
    return;
  }
  if (uploads) {
    const uint64_t t0 = globaltimer_ns();
    while (!atomicAdd(const_cast<uint32_t*>(&sm->mail_a), 0u) && globaltimer_ns() - t0 < kSpinLimitNs) {}
  }
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.spec_flag), "r"((uint32_t)sm->seq) : "memory");
  sm->spec_stage = 2;
}

// Warp 0 builds the FFN plan in shared memory as soon as the loads and
// deferred admissions are final, before the prefetch phase (which only
// touches the prefetch target's state and the copy stream). Item order: the
// shared expert, the speculative plan's routed experts (ascending), the other
// resident hits that are ready (ascending), hits whose (prefetch) upload is
// still in flight by upload id (the copy stream is FIFO), then the demand
// loads and the BA-streamed experts in publication order. Lane l places
// experts l and l + 32 by popcounts over the category masks.
__device__ void build_items(const DecideArgs& a, DecideKSmem* sm) {
  const DevCfg& cfg = sm->cfg;
  const uint32_t B = cfg.B, layer = a.layer;
  const uint32_t lane = (uint32_t)lane_id();
  DecideSmem* d = &sm->d;
  const StepOut& out = d->out;
  Plan* p = &sm->plan;
  EngineState* st = &sm->st;
  LayerState* ls = &sm->ls;
  // residents: lane l takes experts l and l + 32; hit e is out.res[i] with
  // i = its rank in the (ascending) hit set
  const uint64_t res_sel = out.res_mask;
  const uint32_t E = cfg.E;
  const bool v0 = lane < E && ((res_sel >> lane) & 1), v1 = lane + 32 < E && ((res_sel >> (lane + 32)) & 1);
  const uint32_t e0 = lane, e1 = lane + 32;
  // their slots at route time (a deferred admission may since have evicted a hit)
  const int s0 = v0 ? out.res_slot[__popcll(res_sel & ((1ull << e0) - 1))] : -1;
  const int s1 = v1 ? out.res_slot[__popcll(res_sel & ((1ull << e1) - 1))] : -1;
  // uploads already landed (the copy stream is FIFO and copies_done only
  // grows; read during staging): their slots are plain residents again
  const uint32_t landed = sm->landed;
  auto wait_of = [&](int slot) -> uint32_t {
    const uint32_t w = ls->slot_copy[slot];
    if (w && (int32_t)(landed - w) >= 0) {
      ls->slot_copy[slot] = 0;
      return 0;
    }
    return w;
  };
  const uint32_t w0 = v0 ? wait_of(s0) : 0u, w1 = v1 ? wait_of(s1) : 0u;
  const uint64_t spec_m = sm->spec_set;
  const uint64_t wait_m = ballot64(v0 && w0 != 0, v1 && w1 != 0) & ~spec_m;
  const uint64_t ready_m = res_sel & ~wait_m & ~spec_m;
  const uint32_t base = a.shared_w ? 1u : 0u;
  const uint32_t n_spec = (uint32_t)__popcll(spec_m), n_rdy = (uint32_t)__popcll(ready_m);
  const uint32_t n_wait = (uint32_t)__popcll(wait_m);
  __shared__ uint32_t s_wid[kMaxE];
  if (v0) s_wid[e0] = w0;
  if (v1) s_wid[e1] = w1;
  __syncwarp();
  auto item = [&](uint32_t i, const uint16_t* w, uint32_t F, uint32_t wait, uint32_t kind, uint32_t e,
                  uint32_t spec = 0) {
    Item& itm = p->items[i];
    itm.w = w;
    itm.F = F;
    itm.wait = wait;
    itm.kind = kind;
    itm.expert = e;
    itm.spec = spec;
    itm.n_tok = 0;  // token lists are filled in parallel afterwards (fill_items)
  };
  auto place = [&](uint32_t e, int slot, uint32_t w) {
    const uint64_t b = 1ull << e, below = b - 1ull;
    uint32_t i;
    if (spec_m & b) {
      i = base + (uint32_t)__popcll(spec_m & below);
      w = 0;
    } else if (ready_m & b) {
      i = base + n_spec + (uint32_t)__popcll(ready_m & below);
      w = 0;
    } else {
      uint32_t r = 0;  // by upload id (unique)
      for (uint64_t m = wait_m; m; m &= m - 1) r += s_wid[__ffsll((long long)m) - 1] < w;
      i = base + n_spec + n_rdy + r;
    }
    item(i, slot_ptr(a, layer, slot), a.F, w, 1, e);
  };
  if (v0) place(e0, s0, w0);
  if (v1) place(e1, s1, w1);
  if (lane == 0 && a.shared_w) item(0, a.shared_w, a.S, 0, 0, 0);
  const uint32_t n0 = base + n_spec + n_rdy + n_wait;
  for (uint32_t i = lane; i < out.n_load; i += 32)
    item(n0 + i, sm->load_dst[i], a.F, sm->load_id[i], 2, out.load[i], sm->load_spec[i]);
  for (uint32_t i = lane; i < out.n_cpu; i += 32)
    item(n0 + out.n_load + i, sm->cpu_dst[i], a.F, sm->cpu_id[i], 3, out.cpu[i], sm->cpu_spec[i]);
  const uint32_t n_items = n0 + out.n_load + out.n_cpu;
  if (lane == 0) {
    const int8_t* stage_of = sm->stage_of;
    uint32_t n_d2d = 0;
    if (sm->spec_slot >= 0) {  // the speculative buffer -> the admitted cache slot
      p->d2d[n_d2d].src = a.specbuf + (size_t)sm->spec_buf * a.expert_elems;
      p->d2d[n_d2d].dst = slot_ptr(a, layer, sm->spec_slot);
      ++n_d2d;
    }
    for (uint32_t i = 0; i < out.n_def; ++i) {
      const uint32_t e = out.def_e[i];
      const int slot = out.def_slot[i];
      if (stage_of[e] < 0 || slot < 0) continue;
      p->d2d[n_d2d].src = stage_of[e] == kStageSpec ? a.specbuf + (size_t)sm->spec_buf * a.expert_elems
                                                    : a.staging + (size_t)stage_of[e] * a.expert_elems;
      p->d2d[n_d2d].dst = slot_ptr(a, layer, slot);
      ls->slot_copy[slot] = 0;  // filled by this step's FFN epilogue
      ++n_d2d;
    }
    // algorithmic bytes of the FFN launch: every item's weights once, plus
    // u / x in, x out (bf16) and the fp32 layer output
    st->ffn_bytes += 4ull * B * a.d * 2 + (uint64_t)B * a.d * 4 + 3ull * a.S * a.d * 2 +
                     3ull * (n_items - base) * a.F * a.d * 2;
    st->ffn_launches += 1;
    p->n_items = n_items;
    p->n_ready = base + n_spec + n_rdy;
    p->n_spec = sm->spec_n;
    p->n_local = n0;
    p->n_d2d = n_d2d;
    p->d2d_elems = a.expert_elems;
    p->seq = (uint32_t)sm->seq;
  }
  __syncwarp();
}

// The prefetch upload commands (mailbox entry B), after the prefetch phase.
__device__ void build_prefetch_cmds(const DecideArgs& a, DecideKSmem* sm, uint32_t wait_ffn);

// Predictor mode: mailbox entry B of the PREVIOUS step (its schedule_prefetch
// ran at the start of this step), before this step's entry A. Warp 0.
__device__ void EarlyPublish::prefetched(DecideSmem*) const {
  if (lane_id() == 0 && sm->seq >= 2) {
    const DecideArgs& A = *a;
    build_prefetch_cmds(A, sm, (uint32_t)(sm->seq - 1));
    const uint64_t mseq = 2 * (sm->seq - 1);
    wait_ring_slot(A, mseq, &sm->st.ack_cache);
    MailEntry* me = &A.ring[mseq % kRing];
    const uint32_t nc = sm->n_cmds;
    for (uint32_t i = 0; i < nc; ++i) put_wire(&me->cmd[i], sm->cmd[i], mseq);
    me->n = nc;
    me->seq = (mseq << 8) | nc;
    sm->n_cmds = 0;
  }
  __syncwarp();
}

__device__ void build_prefetch_cmds(const DecideArgs& a, DecideKSmem* sm, uint32_t wait_ffn) {
  const uint32_t E = sm->cfg.E, layer = a.layer;
  const StepOut& out = sm->d.out;
  EngineState* st = &sm->st;
  uint32_t n_cmds = 0;
  for (uint32_t i = 0; i < out.n_pref; ++i) {
    const uint32_t e = out.pref[i];
    const int slot = out.pref_slot[i];
    const uint32_t tlayer = out.pref_layer;
    uint16_t* dst = slot >= 0 ? slot_ptr(a, tlayer, slot) : a.staging;
    const uint32_t id = ++st->next_copy;
    MailCmd& c = sm->cmd[n_cmds++];
    c.src_off = ((uint64_t)tlayer * E + e) * a.expert_elems * 2;
    c.dst = (uint64_t)dst;
    c.bytes = a.expert_elems * 2;
    c.id = id;
    c.wait_ffn = wait_ffn;
    c.kind = 0;
    c.gen = c.buf = c.pad = 0;
    LayerState* tls = (tlayer == layer) ? &sm->ls : &sm->tls;
    if (slot >= 0) tls->slot_copy[slot] = id;
  }
  sm->n_cmds = n_cmds;
}

// Warp 0, as soon as the step's FFN items are final (before the prefetch
// phase): build the plan, fill token lists / weights, publish it to global
// memory and (speculative mode) release it to the running FFN kernel.
__device__ void fill_items(const DecideArgs& a, DecideKSmem* sm);

__device__ void EarlyPublish::plan_ready(DecideSmem* d) const {
  const DecideArgs& A = *a;
  const int lane = lane_id();
  const uint32_t B = sm->cfg.B;
  if ((uint32_t)lane < B) {  // combine-weight denominators (Mixtral renormalisation)
    const uint32_t t = lane;
    float s = 0.f;
    for (uint32_t i = 0; i < d->nsel[t]; ++i) s += sm->sc[t][d->sel[t][i]];
    sm->denom[t] = s;
  }
  __syncwarp();
#ifdef MOEB_PROFILE_PHASES
  uint64_t tq = ptimer();
  auto pmark = [&](int i) { if (lane == 0) { const uint64_t n = ptimer(); sm->st.prof[i] += n - tq; tq = n; } };
#else
  auto pmark = [](int) {};
#endif
  build_items(A, sm);
  pmark(24);
  fill_items(A, sm);
  __syncwarp();
  pmark(25);
  Plan* gp = A.plan;
  const uint32_t n_items = sm->plan.n_items;
  const uint64_t* src = reinterpret_cast<const uint64_t*>(&sm->plan);
  uint64_t* dst = reinterpret_cast<uint64_t*>(gp);
  const size_t words = (offsetof(Plan, items) + n_items * sizeof(Item)) / 8;
  for (uint32_t i = lane; i < words; i += 32) dst[i] = src[i];
  const size_t d0 = offsetof(Plan, d2d) / 8, d1 = d0 + sm->plan.n_d2d * sizeof(D2D) / 8;
  for (uint32_t i = d0 + lane; i < d1; i += 32) dst[i] = src[i];
  pmark(26);
  if (A.spec_plan) {
    // the FFN kernel (already running its speculative items) takes the final
    // plan from this flag instead of waiting for this kernel to complete:
    // every writer fences, then one release
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(A.spec_flag + 1), "r"((uint32_t)sm->seq) : "memory");
      if (A.tl) A.tl[12] = globaltimer_ns();
    }
  }
  __syncwarp();
  pmark(27);
}

// Token lists and combine weights of every plan item: lane t holds token t's
// selection mask, one ballot per item gives its tokens (ascending) and each
// selecting lane writes its own entry.
__device__ void fill_items(const DecideArgs& a, DecideKSmem* sm) {
  const uint32_t B = sm->cfg.B;
  const uint32_t lane = (uint32_t)lane_id();
  const DecideSmem* d = &sm->d;
  Plan* p = &sm->plan;
  uint64_t selm = 0;
  if (lane < B)
    for (uint32_t i = 0; i < d->nsel[lane]; ++i) selm |= 1ull << d->sel[lane][i];
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t ii = 0; ii < p->n_items; ++ii) {
    Item& itm = p->items[ii];
    const uint32_t kind = itm.kind, e = itm.expert;
    const bool sel = lane < B && (kind == 0 || ((selm >> e) & 1));
    const uint32_t toks = __ballot_sync(0xffffffffu, sel);
    if (sel) {
      float wt;
      if (kind == 0) {
        wt = a.shared_gate ? sm->sg[lane] : 1.0f;
      } else {
        wt = sm->sc[lane][e];
        if (a.renormalize) wt = __fdiv_rn(wt, sm->denom[lane]);
        wt = __fmul_rn(wt, a.routed_scale);
      }
      const uint32_t pos = __popc(toks & lt);
      itm.tok[pos] = (uint8_t)lane;
      itm.wt[pos] = wt;
    }
    if (lane == 0) itm.n_tok = __popc(toks);
  }
  __syncwarp();
}

// Router gate (all CTAs) then, in the last CTA to finish, the decision step,
// the FFN plan and the upload mailbox. One launch per layer.
__global__ void __launch_bounds__(kGdThreads, 1) gate_decide_kernel(GateDecideArgs ga) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
#ifdef MOEB_PROFILE_PHASES
#define MOEB_T(x) const uint64_t x = gtimer()
#else
#define MOEB_T(x) const uint64_t x = 0
#endif
  // the gate CTAs' router rows first (static weights: the load overlaps the
  // previous layer's FFN tail); then PDL: wait for the previous layer's FFN
  // (x, plan buffers), and let the next kernel's CTAs start launching as ours retire
  GateWPre wpre;
  wpre.ok = false;
  if (blockIdx.x != 0) wpre = gate_w_prefetch(ga.g, blockIdx.x - 1);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  MOEB_T(t_entry);
  __shared__ uint64_t t_plan_g_s;
  uint64_t& t_plan_g = t_plan_g_s;
#ifdef MOEB_PROFILE_PHASES
  if (threadIdx.x == 0) atomicMin(reinterpret_cast<unsigned long long*>(&ga.d.st->prof[14]), (unsigned long long)t_entry);
#endif
  // CTAs 1..G: the router gate (RMSNorm + GEMV rows); CTA 0: the decision.
  // The decider stages the step's state while the gate runs, then waits for
  // the gate CTAs' arrivals (they are few and co-resident) instead of the
  // last gate CTA electing itself after the fact.
  const uint32_t n_gate = gridDim.x - 1;
  if (blockIdx.x != 0) {
    // us [B][d] bf16 aliases the decision workspace
    gate_phase(ga.g, reinterpret_cast<uint16_t*>(smem_raw), blockIdx.x - 1, n_gate, ga.g.x, ga.g.logits, true, &wpre);
    if (ga.g.x_pred) {
      // the predictor: this layer's router on the previous layer's partial
      // forward (shared expert + resident hits)
      __syncthreads();
      gate_phase(ga.g, reinterpret_cast<uint16_t*>(smem_raw), blockIdx.x - 1, n_gate, ga.g.x_pred, ga.g.plogits,
                 false);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ga.ticket, 1u);
    }
    return;
  }
  DecideKSmem* sm = reinterpret_cast<DecideKSmem*>(smem_raw);
  const DecideArgs& a = ga.d;
  if (a.tl && threadIdx.x == 0) a.tl[3] = globaltimer_ns();
  // the FFN grid counters of this step, zeroed before the FFN kernel (which
  // may already be resident) can see the speculative plan or the final one:
  // fenced before the barrier that precedes both releases
  // (by the last warp: its fence does not delay warp 0's staging loads)
  if (threadIdx.x >= blockDim.x - 32) {
    for (uint32_t i = threadIdx.x - (blockDim.x - 32); i < (uint32_t)kFfnCtrWords; i += 32) a.ffn_ctr[i] = 0;
    __threadfence();
  }
  const int warp = warp_id(), lane = lane_id();
  const uint32_t nw = blockDim.x >> 5;
  // stage the step's state: one parallel load phase (it / seq come from the
  // host, so every address is known at launch)
  const uint32_t L = a.cfg.L, B = a.cfg.B, E = a.cfg.E, layer = a.layer;
  const uint64_t it = a.it;
  uint32_t tl = layer + 1;
  uint64_t tit = it;
  if (tl == L) { tl = 0; ++tit; }
  const bool has_target = tit < a.total_iters;
  const bool want_next = a.cfg.pre && has_target && a.trace;
  const bool smem_hist = a.cfg.window * E <= kMaxHistSmem;
  const size_t hwords = (size_t)a.cfg.window * E;
  {
    // every staging load is issued before any store: one memory latency
    static_assert(sizeof(EngineState) / 8 <= kGdThreads && sizeof(LayerState) / 8 <= kGdThreads, "staging");
    constexpr uint32_t kStW = sizeof(EngineState) / 8, kLsW = sizeof(LayerState) / 8;
    constexpr int kHw = kMaxHistSmem / kGdThreads;  // ring words per thread
    const uint32_t tid = threadIdx.x;
    const bool two = want_next && tl != layer;
    const uint64_t* g_st = reinterpret_cast<const uint64_t*>(a.st);
    const uint64_t* g_ls = reinterpret_cast<const uint64_t*>(&a.layers[layer]);
    const uint64_t* g_tls = reinterpret_cast<const uint64_t*>(&a.layers[tl]);
    const uint64_t* g_h = reinterpret_cast<const uint64_t*>(a.hist + layer * hwords);
    const uint64_t* g_th = reinterpret_cast<const uint64_t*>(a.hist + tl * hwords);
    uint64_t r_st = 0, r_ls = 0, r_tls = 0, r_h[kHw], r_th[kHw];
    const uint32_t r_cd = 0;
    if (tid < kStW) r_st = g_st[tid];
    if (tid < kLsW) r_ls = g_ls[tid];
    if (two && tid < kLsW) r_tls = g_tls[tid];
    if (smem_hist) {
#pragma unroll
      for (int k = 0; k < kHw; ++k) {
        const uint32_t i = tid + k * kGdThreads;
        if (i < hwords) {
          r_h[k] = g_h[i];
          if (two) r_th[k] = g_th[i];
        }
      }
    }
    if (tid < kStW) reinterpret_cast<uint64_t*>(&sm->st)[tid] = r_st;
    if (tid < kLsW) reinterpret_cast<uint64_t*>(&sm->ls)[tid] = r_ls;
    if (two && tid < kLsW) reinterpret_cast<uint64_t*>(&sm->tls)[tid] = r_tls;
    if (smem_hist) {
#pragma unroll
      for (int k = 0; k < kHw; ++k) {
        const uint32_t i = tid + k * kGdThreads;
        if (i < hwords) {
          reinterpret_cast<uint64_t*>(sm->hist)[i] = r_h[k];
          if (two) reinterpret_cast<uint64_t*>(sm->thist)[i] = r_th[k];
        }
      }
    }
    if (threadIdx.x == 0) sm->cfg = a.cfg;
    (void)r_cd;
  }
  // trace-driven routing: this layer's logits (and the next layer's, for
  // the predictor) come from the trace, not the gate — staged now, while the
  // gate CTAs run, and normalised in place after the gate arrivals
  if (a.trace) {
    const float* tr = a.trace + ((it % a.trace_steps) * L + layer) * B * E;
    const float* ntr = a.trace + ((tit % a.trace_steps) * L + tl) * B * E;
    for (uint32_t i = threadIdx.x; i < B * E; i += blockDim.x) {
      const float v = __ldg(tr + i);
      const float nv = want_next ? __ldg(ntr + i) : 0.f;
      sm->sc[i / E][i % E] = v;
      if (want_next) sm->nsc[i / E][i % E] = nv;
    }
  }
  MOEB_T(t_staged0);
  // the router logits and u of this layer: every gate CTA has arrived
  if (threadIdx.x == 0) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_u32(ga.ticket) < n_gate) {
      if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 7u); break; }
    }
    *ga.ticket = 0;  // reset for the next layer (ordered by this kernel's completion)
    sm->landed = *reinterpret_cast<const volatile uint32_t*>(a.copies_done);
  }
  __syncthreads();
  MOEB_T(t_gate);
  const uint32_t jobs = want_next ? 2 * B : B;
  for (uint32_t j = warp; j < jobs; j += nw) {
    if (j < B) {
      const uint32_t t = j;
      const float* lg = a.trace ? sm->sc[t] : a.logits + (size_t)t * (E + 1);  // in place for the trace
      softmax_warp(lg, E, sm->sc[t]);
      if (lane == 0 && a.shared_gate) {
        const float z = a.logits[(size_t)t * (E + 1) + E];
        sm->sg[t] = __fdiv_rn(1.0f, 1.0f + expf(-z));
      }
    } else {
      const uint32_t t = j - B;
      softmax_warp(sm->nsc[t], E, sm->nsc[t]);
    }
  }
  // the shared expert depends on nothing the decision computes: released to
  // the (already resident) FFN right after the gate, before classification,
  // by the last warp beside the softmax (batch 1: warp 0). The release store
  // orders this thread's item writes (no separate fence).
  if (a.shared_first && threadIdx.x == blockDim.x - 32) {
    Item& it0 = a.spec_plan->items[0];
    it0.w = a.shared_w;
    it0.F = a.S;
    it0.wait = 0;
    it0.n_tok = 1;
    it0.kind = 0;
    it0.expert = 0;
    it0.tok[0] = 0;
    it0.wt[0] = a.shared_gate ? __fdiv_rn(1.0f, 1.0f + expf(-a.logits[E])) : 1.0f;  // = sg[0]
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.spec_flag + 2), "r"((uint32_t)a.seq) : "memory");
  }
  const bool run_pending = a.predictor && sm->st.pf_pending && sm->st.pf_layer == layer && sm->st.pf_it == it;
  if (run_pending)  // the prediction for this layer: softmax of the router on the partial forward
    for (uint32_t t = warp; t < B; t += nw) softmax_warp(a.plogits + (size_t)t * (E + 1), E, sm->nsc[t]);
  if (threadIdx.x == 0) {
    sm->it = it;
    sm->seq = a.seq;
    sm->mail_a = 0;
    sm->spec_stage = 0;
    sm->d.next_has_pred = run_pending ? (B >= 64 ? ~0ull : (1ull << B) - 1ull) : 0ull;
  }
  __syncthreads();
  const DevCfg& cfg = sm->cfg;
  for (uint32_t i = threadIdx.x; i < B * E; i += blockDim.x) {
    const uint32_t t = i / E, e = i % E;
    sm->d.s[t][e] = (double)sm->sc[t][e];
    if (want_next) sm->d.ns[t][e] = (double)sm->nsc[t][e];
    if (run_pending) sm->d.np[t][e] = (double)sm->nsc[t][e];
    if (a.scores_log && a.seq <= a.rec_cap) a.scores_log[((a.seq - 1) * B + t) * E + e] = sm->sc[t][e];
    if (run_pending && a.pred_log && a.seq <= a.rec_cap) a.pred_log[((a.seq - 1) * B + t) * E + e] = sm->nsc[t][e];
  }
  __syncthreads();
  MOEB_T(t_staged);

  StepCtx cx;
  cx.cfg = &cfg;
  cx.st = &sm->st;
  cx.ls = &sm->ls;
  cx.hist_l = smem_hist ? sm->hist : a.hist + layer * hwords;
  cx.tls = (tl == layer) ? &sm->ls : &sm->tls;
  cx.thist = (tl == layer) ? cx.hist_l : (smem_hist ? sm->thist : a.hist + tl * hwords);
  cx.logs = nullptr;
  cx.it = it;
  cx.layer = layer;
  cx.has_target = (want_next || (a.predictor && has_target)) ? 1u : 0u;
  cx.target_layer = tl;
  cx.target_it = tit;
  cx.prof = sm->st.prof;
  cx.defer_prefetch = a.predictor;
  cx.f32_scores = 1;  // softmax in fp32, widened
  cx.run_pending = run_pending;
  cx.prev_rec = (a.recs && sm->seq >= 2 && sm->seq - 1 <= a.rec_cap) ? a.recs + (sm->seq - 2) : nullptr;
  StepRec* rec = nullptr;
  TokRec* toks = nullptr;
  if (a.recs && sm->seq <= a.rec_cap) {
    rec = a.recs + (sm->seq - 1);
    toks = a.toks + (sm->seq - 1) * B;
  }
  decide_step(cx, &sm->d, &sm->n, &sm->s, rec, toks, EarlyPublish{&a, sm});
  __syncthreads();
  MOEB_T(t_decided);

  if (threadIdx.x == 0) {
    // predictor mode: entry B of this step is published by the next step
    if (!a.predictor) build_prefetch_cmds(a, sm, (uint32_t)sm->seq);
    else sm->n_cmds = 0;
    // speculative upload for the next step: the first expert of the prefetch
    // queue's ranking that is still not resident in the target layer after
    // this step's prefetches (the reference's predictor, prefetch.cpp:34-115;
    // its virtual clock decides what is ADMITTED, this only moves bytes early)
    if (a.spec_up && !a.predictor && want_next) {
      const LayerState* tls = (tl == layer) ? &sm->ls : &sm->tls;
      uint32_t cand = 0xffffffffu;
      for (uint32_t r = 0; r < E; ++r)
        if (!((tls->mask >> sm->d.qorder[r]) & 1ull)) { cand = sm->d.qorder[r]; break; }
      const uint32_t b = (uint32_t)((sm->seq + 1) & 1);
      if (cand != 0xffffffffu) {
        EngineState* st = &sm->st;
        const uint32_t gen = ++st->sp_gen_next;
        st->sp_valid[b] = 1;
        st->sp_layer[b] = tl;
        st->sp_it[b] = tit;
        st->sp_expert[b] = cand;
        st->sp_gen[b] = gen;
        st->sp_jobs += 1;
        MailCmd& c = sm->cmd[sm->n_cmds++];
        c.src_off = ((uint64_t)tl * E + cand) * a.expert_elems * 2;
        c.dst = (uint64_t)(a.specbuf + (size_t)b * a.expert_elems);
        c.bytes = a.expert_elems * 2;
        c.id = 0;
        c.wait_ffn = 0;
        c.kind = 1;
        c.gen = gen;
        c.buf = b;
        c.pad = 0;
      } else {
        sm->st.sp_valid[b] = 0;
      }
    }
    // entry B's ring slot must have been consumed by the copy thread
    if (!a.predictor) wait_ring_slot(a, 2 * sm->seq, &sm->st.ack_cache);
    sm->st.seq = sm->seq;
    if (layer == L - 1) sm->st.it = it + 1;
  }
  if (threadIdx.x == 0) {
    MOEB_T(t_plan);
    t_plan_g = t_plan;
#ifdef MOEB_PROFILE_PHASES
    sm->st.prof[0] += t_gate - t_staged0;   // waiting for the gate CTAs after staging
    sm->st.prof[1] += t_staged0 - t_entry;  // staging (overlaps the gate)
    sm->st.prof[2] += t_staged - t_gate;    // softmax + scores
    sm->st.prof[3] += t_decided - t_staged;
    sm->st.prof[9] += t_plan - t_decided;
#endif
    (void)t_entry; (void)t_gate; (void)t_staged0; (void)t_staged; (void)t_decided; (void)t_plan;
  }
  __syncthreads();
  // publish: prefetch commands -> mapped host ring, state write-back (the
  // plan went out in EarlyPublish::plan_ready)
  {
    if (!a.predictor) {
      MailEntry* me = &a.ring[(2 * sm->seq) % kRing];
      const uint32_t nc = sm->n_cmds;
      for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) put_wire(&me->cmd[i], sm->cmd[i], 2 * sm->seq);
      if (threadIdx.x == 0) me->n = nc;
    }
    cta_copy(a.st, &sm->st);
    cta_copy(&a.layers[layer], &sm->ls);
    if (want_next && tl != layer) cta_copy(&a.layers[tl], &sm->tls);
    if (smem_hist)
      for (uint32_t i = threadIdx.x; i < hwords; i += blockDim.x) a.hist[layer * hwords + i] = sm->hist[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    MOEB_T(t_pub0);
    const uint32_t nc = sm->n_cmds;
    if (!a.predictor) a.ring[(2 * sm->seq) % kRing].seq = ((2 * sm->seq) << 8) | nc;
    if (a.tl) a.tl[5] = globaltimer_ns();
#ifdef MOEB_PROFILE_PHASES
    const uint64_t t_pub1 = gtimer();
    a.st->prof[10] += t_pub1 - t_pub0;
    a.st->prof[12] += t_pub0 - t_plan_g;
    const uint64_t first = a.st->prof[14];
    a.st->prof[15] += t_entry - first;       // start skew of the deciding CTA
    a.st->prof[11] += t_pub1 - first;        // first CTA start -> publish done
    a.st->prof[14] = ~0ull;
#endif
    (void)t_pub0;
  }
  // warm L2 with the next layer's state (the FFN streams ~140 MB of weights
  // through L2 with evict-first in between): layer state, score ring, and
  // the next routing logits row
  {
    const uint32_t nl = tl, nl2 = (tl + 1 == L) ? 0 : tl + 1;
    const char* regions[3] = {reinterpret_cast<const char*>(&a.layers[nl]),
                              reinterpret_cast<const char*>(a.hist + nl * hwords),
                              reinterpret_cast<const char*>(&a.layers[nl2])};
    const uint32_t sizes[3] = {(uint32_t)sizeof(LayerState), (uint32_t)(hwords * 8), (uint32_t)sizeof(LayerState)};
    uint32_t line = threadIdx.x;
    for (int r = 0; r < 3; ++r) {
      const uint32_t nlines = (sizes[r] + 127) / 128;
      if (line < nlines) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(regions[r] + line * 128));
        break;
      }
      line -= nlines;
    }
    if (a.trace && threadIdx.x < 2) {
      const uint64_t nit = (tl == 0) ? it + 1 : it;
      const float* row = a.trace + (((nit % a.trace_steps) * L + tl) * B) * E;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(row) + threadIdx.x * 128));
    }
  }
}

// =================================================================== host

struct IoAcc {
  uint64_t h2d_bytes = 0, h2d_copies = 0, d2d_copies = 0, steps = 0;
  double copy_ms = 0.0;     // speculative chunks (every one timed)
  double upload_ms = 0.0;   // the timed uploads (one in copy_every)
  uint64_t timed_uploads = 0;
  uint64_t spec_jobs = 0, spec_promoted = 0, spec_chunks = 0, spec_bytes = 0;
  std::vector<float> per_copy_ms;  // first 65536 uploads since the last reset (moeb_get_copy_times)
};

}  // namespace moeb

using namespace moeb;

struct moeb_stack {
  moeb_config cfg{};
  moeb_model model{};
  DevCfg dcfg{};
  int device = 0;
  uint32_t L = 0, E = 0, B = 0, d = 0, F = 0, S = 0, slots_alloc = 0, n_stage = 0;
  uint64_t expert_elems = 0;
  DevBuf<uint16_t> gate_w, shared_w, sgate_w, slots, staging, hidden, u;
  DevBuf<float> logits, h, y_layers, trace, scores_log;
  // predictor mode (MOEB_MODEL_PREDICTOR): partial forward, its router
  // logits, the predictions used per step
  bool predictor = false;
  // speculative uploads (split-K stacks with stage Pre and a logits trace):
  // two expert-sized buffers, their landed generations, the copy thread's jobs
  bool spec_up = false;
  DevBuf<uint16_t> specbuf;
  DevBuf<uint32_t> spec_done;
  struct SpecJob {
    uint32_t gen = 0, chunks = 0, next = 0;  // next: chunks issued so far
    uint64_t src_off = 0, dst = 0, bytes = 0;
    bool live = false;
  } sjob[2];
  cudaEvent_t ev_spec = nullptr, ev_dem = nullptr;  // last speculative chunk / last upload issued
  bool spec_inflight = false, dem_inflight = false;
  DevBuf<uint16_t> xpred;
  DevBuf<float> plogits, pred_log;
  DevBuf<EngineState> st;
  DevBuf<LayerState> layers;
  DevBuf<double> hist;
  DevBuf<Plan> plan, spec_plan;
  DevBuf<uint32_t> spec_flag;
  bool spec = false;
  bool splitk = false;  // batch-1 split-K FFN; experts stored row-interleaved [F][3][d]
  bool umma = false;    // batched tensor-core FFN (ffn_umma.cuh); experts stored UMMA-tiled
  UmLaunch um{};
  DevBuf<uint16_t> xt;  // activations, SW128-tiled (umma)
  DevBuf<float> part;   // partial outputs per (item, down split) (umma)
  DevBuf<float> gpart;  // gate_up K-split partials (umma)
  DevBuf<uint32_t> gcnt;
  uint32_t layout_flags() const { return splitk ? MOEB_MODEL_DOWN_T : umma ? MOEB_MODEL_TILED : 0u; }
  uint32_t unit_rows = 0, ffn_dbg = 0;
  bool sk_shared_prefetch = true;  // split-K: shared-expert rows issued before the release (MOEB_NO_SHARED_PREFETCH=1: off)
  DevBuf<uint32_t> ffn_ctr, copies_done, ffn_done;
  DevBuf<uint64_t> ffn_ts;  // MOEB_FFN_TSTAMP: per-CTA phase stamps of the last split-K FFN launch
  DevBuf<StepRec> recs;
  DevBuf<uint64_t> timeline;  // [rec_cap][kTlWords] (MOEB_MODEL_TRACE_TIMELINE)
  DevBuf<TokRec> toks;
  uint64_t rec_cap = 0;
  uint64_t trace_steps = 0, total_iters = ~0ull;
  uint16_t* pool = nullptr;
  bool own_pool = false, registered_pool = false;
  MailEntry* ring = nullptr;
  uint64_t* ack = nullptr;
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  std::thread copier;
  std::atomic<bool> stop{false};
  std::atomic<int> copier_error{0};
  std::string copier_msg;
  int ffn_grid = 0;
  FfnLaunch ffn{};
  size_t gd_smem = 0;
  DevBuf<uint32_t> ticket;
  MailEntry* ring_dev = nullptr;
  uint64_t* ack_dev = nullptr;
  uint64_t host_it = 0, host_seq = 0;  // mirrors of EngineState::it / seq
  // Serial (profiler-safe) mode: upload dependencies are stream waits on the
  // compute stream (cuStreamWaitValue32) set up by the host after each decide
  // kernel, never in-kernel spins on a concurrently running engine. Chosen
  // with MOEB_SERIAL=1 or automatically under ncu / nsys / compute-sanitizer,
  // which serialise kernels (and the copy thread's API calls) behind the one
  // being measured, so an FFN spinning on copies_done could never see them.
  // Prefill (moeb_prefill): buffers sized for pf_cap tokens; staging for the
  // non-resident experts of two layers (the layer being computed and the next
  // one, uploading); a copy stream and its events.
  uint32_t pf_cap = 0, pf_R = 0, pf_tiles = 0;
  DevBuf<uint16_t> pf_u, pf_hid, pf_stage, pf_tiled;
  DevBuf<float> pf_logits, pf_scores, pf_wts, pf_slot_w, pf_out;
  DevBuf<uint8_t> pf_sel;
  DevBuf<int32_t> pf_entry;
  DevBuf<uint32_t> pf_cnt, pf_cursor;
  DevBuf<PfItem> pf_items;
  DevBuf<PfHdr> pf_hdr;
  DevBuf<uint32_t> pf_ctr;
  DevBuf<unsigned char> pf_xg, pf_hg;
  cudaStream_t pf_copy = nullptr;
  cudaEvent_t pf_up[2] = {}, pf_free[2] = {};
  // MOEB_MODEL_LOG_STEPS: the last prefill's per-layer inputs, scores,
  // selections and fp32 outputs (moeb_get_prefill_log)
  uint32_t pf_log_n = 0, pf_last_n = 0;
  DevBuf<uint16_t> pf_log_x;
  DevBuf<float> pf_log_scores, pf_log_y;
  DevBuf<uint8_t> pf_log_sel;
  bool serial = false, serial_at_create = false;
  uint32_t serial_need = 0;  // highest upload id the next FFN may depend on
  uint64_t n_launch_layers = 0;        // (gate+decide, FFN) launch pairs
  std::mutex io_mu;
  IoAcc io;
  static constexpr int kEv = 512;
  cudaEvent_t ev_a[kEv] = {}, ev_b[kEv] = {};
  bool ev_live[kEv] = {};
  bool ev_chunk[kEv] = {};
  int ev_next = 0;

  // Kernel timing (MOEB_MODEL_TIME_KERNELS): 3 events per layer on the
  // compute stream: before gate+decide, before FFN, after FFN.
  bool timing = false;
  static constexpr int kTk = 3 * 1024;
  cudaEvent_t tk_ev[kTk] = {};
  int tk_n = 0;       // recorded, not yet harvested
  int tk_head = 0;    // oldest unharvested
  int tk_phase = 0;
  double kern_ms[2] = {0, 0};  // gate+decide, ffn
  uint64_t kern_n[2] = {0, 0};
  void tk_harvest_one() {
    const int i0 = tk_head;
    cudaEventSynchronize(tk_ev[(i0 + 2) % kTk]);
    for (int k = 0; k < 2; ++k) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, tk_ev[(i0 + k) % kTk], tk_ev[(i0 + k + 1) % kTk]) == cudaSuccess) {
        kern_ms[k] += ms;
        kern_n[k] += 1;
      }
    }
    tk_head = (tk_head + 3) % kTk;
    tk_n -= 3;
  }
  void tick(cudaStream_t s) {
    if (tk_phase == 0 && tk_n + 3 > kTk) tk_harvest_one();
    cudaEventRecord(tk_ev[(tk_head + tk_n) % kTk], s);
    ++tk_n;
    tk_phase = (tk_phase + 1) % 3;
  }
  void tk_harvest_all() {
    while (tk_n >= 3) tk_harvest_one();
  }

  void harvest(int i) {  // requires io_mu
    if (!ev_live[i]) return;
    cudaEventSynchronize(ev_b[i]);
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ev_a[i], ev_b[i]) == cudaSuccess) {
      if (ev_chunk[i]) {
        io.copy_ms += ms;
      } else {
        io.upload_ms += ms;
        io.timed_uploads += 1;
        if (io.per_copy_ms.size() < 65536) io.per_copy_ms.push_back(ms);
      }
    }
    ev_live[i] = false;
    ev_chunk[i] = false;
  }

  // Harvest the oldest live copy-event pair if it has completed (idle loop;
  // a non-blocking query, so the poller stays responsive).
  void harvest_some() {
    for (int n = 0; n < 4; ++n) {  // the oldest slots: the next ones to be reused
      const int i = (ev_next + n) % kEv;
      if (!ev_live[i]) continue;
      if (cudaEventQuery(ev_b[i]) != cudaSuccess) return;
      std::lock_guard<std::mutex> g(io_mu);
      harvest(i);
      return;
    }
  }

  // Expert sources (moeb_set_expert_sources): per (layer, expert) a device
  // pointer to the expert's weights in some GPU's HBM (a peer GPU's over
  // NVLink, or this one's) instead of the pinned host pool. Empty: host pool.
  std::vector<const char*> src_tab;
  const char* upload_src(uint64_t src_off) const {
    if (src_tab.empty()) return reinterpret_cast<const char*>(pool) + src_off;
    const uint64_t eb = expert_elems * 2;
    return src_tab[src_off / eb] + src_off % eb;
  }
  // one upload: the copy, then copies_done := id (the FFN waits on it).
  // One upload in copy_every is bracketed by timing events (their two
  // event records delay the copy's start by a few us: on the bench workload,
  // same box, timing every upload 7.69 ms/token, one in 8 7.66, none 7.62-7.65);
  // the copy-stream busy time is extrapolated from the timed ones (all
  // uploads are one expert). MOEB_COPY_TIMING_EVERY=n (1: every upload, 0: none).
  const uint32_t copy_every = [] {
    const char* v = getenv("MOEB_COPY_TIMING_EVERY");
    return v ? (uint32_t)atoi(v) : 8u;
  }();
  void issue_upload(const MailCmd& c, CUdeviceptr done_ptr) {
    if (copy_every == 0 || io.h2d_copies % copy_every != 0) {  // untimed: the copy and its signal only
      const cudaError_t ce = cudaMemcpyAsync(reinterpret_cast<void*>(c.dst), upload_src(c.src_off), c.bytes,
                                             cudaMemcpyDefault, copy_stream);
      if (p_write32(copy_stream, done_ptr, c.id, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS || ce != cudaSuccess) {
        copier_msg = "upload failed";
        copier_error = 5;
      }
      std::lock_guard<std::mutex> g(io_mu);
      io.h2d_bytes += c.bytes;
      io.h2d_copies += 1;
      return;
    }
    // submit first, account after: the copy's start is what the GPU waits for
    const int ei = ev_next;
    ev_next = (ev_next + 1) % kEv;
    if (ev_live[ei]) {  // normally harvested while the thread idled (harvest_some)
      std::lock_guard<std::mutex> g(io_mu);
      harvest(ei);
    }
    cudaEventRecord(ev_a[ei], copy_stream);
    const cudaError_t ce = cudaMemcpyAsync(reinterpret_cast<void*>(c.dst), upload_src(c.src_off), c.bytes,
                                           cudaMemcpyDefault, copy_stream);
    if (p_write32(copy_stream, done_ptr, c.id, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) {
      copier_msg = "cuStreamWriteValue32 failed";
      copier_error = 5;
    }
    cudaEventRecord(ev_b[ei], copy_stream);
    if (ce != cudaSuccess) {
      copier_msg = std::string("upload failed: ") + cudaGetErrorString(ce);
      copier_error = 5;
    }
    std::lock_guard<std::mutex> g(io_mu);
    ev_live[ei] = true;
    io.h2d_bytes += c.bytes;
    io.h2d_copies += 1;
  }

  // Speculative uploads move in chunks so a real upload never queues behind
  // more than one chunk: a chunk is issued only while the copy stream has no
  // upload and no other chunk in flight. The last chunk sets spec_done[buf].
  static constexpr uint32_t kSpecChunks = 16;  // ~1.1 MB, ~20 us each for a DSV2-Lite expert
  void issue_spec_chunk(uint32_t b) {
    SpecJob& j = sjob[b];
    const uint64_t per = (j.bytes / j.chunks + 255) & ~255ull;
    const uint64_t off = (uint64_t)j.next * per;
    const uint64_t n = off < j.bytes ? std::min(per, j.bytes - off) : 0;
    const int ei = ev_next;
    ev_next = (ev_next + 1) % kEv;
    if (ev_live[ei]) {
      std::lock_guard<std::mutex> g(io_mu);
      harvest(ei);
    }
    cudaEventRecord(ev_a[ei], copy_stream);
    const cudaError_t ce = cudaMemcpyAsync(reinterpret_cast<void*>(j.dst + off), upload_src(j.src_off + off), n,
                                           cudaMemcpyDefault, copy_stream);
    cudaEventRecord(ev_b[ei], copy_stream);
    if (ce != cudaSuccess) {
      copier_msg = std::string("speculative upload failed: ") + cudaGetErrorString(ce);
      copier_error = 5;
    }
    j.next += 1;
    if (j.next == j.chunks) {
      if (p_write32(copy_stream, (CUdeviceptr)(spec_done.p + b), j.gen, CU_STREAM_WRITE_VALUE_DEFAULT) !=
          CUDA_SUCCESS) {
        copier_msg = "cuStreamWriteValue32 failed";
        copier_error = 5;
      }
      j.live = false;
    }
    std::lock_guard<std::mutex> g(io_mu);
    ev_live[ei] = true;
    ev_chunk[ei] = true;  // copy-engine busy time, not a whole-expert upload
    io.spec_chunks += 1;
    io.spec_bytes += n;
    io.h2d_bytes += n;
  }

  // a command of mailbox entry mseq, once all six words carry its tag
  // (WireCmd); the stores reach host memory in any order
  MailCmd take_cmd(const WireCmd* wc, uint64_t mseq) {
    const uint64_t t = wire_tag(mseq), hi = ~((1ull << 48) - 1);
    uint64_t w[6];
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned spin = 0;; ++spin) {
      bool ok = true;
      for (int j = 0; j < 6; ++j) {
        w[j] = reinterpret_cast<const volatile uint64_t*>(wc->w)[j];
        ok &= (w[j] & hi) == t;
      }
      if (ok) break;
      __builtin_ia32_pause();
      if ((spin & 1023u) == 1023u && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(5)) {
        copier_msg = "mailbox command words did not arrive";
        copier_error = 5;
        return MailCmd{};
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const uint64_t m = (1ull << 48) - 1;
    MailCmd c{};
    c.src_off = w[0] & m;
    c.dst = w[1] & m;
    c.bytes = w[2] & ((1ull << 40) - 1);
    c.kind = (uint32_t)(w[2] >> 40) & 15u;
    c.buf = (uint32_t)(w[2] >> 44) & 15u;
    c.id = (uint32_t)w[3];
    c.wait_ffn = (uint32_t)w[4];
    c.gen = (uint32_t)w[5];
    return c;
  }

  void copy_loop() {
    cudaSetDevice(device);
    CUdeviceptr done_ptr = (CUdeviceptr)copies_done.p;
    CUdeviceptr ffn_ptr = (CUdeviceptr)ffn_done.p;
    uint64_t expect = 1;
    unsigned spins = 0;
    auto t_poll = std::chrono::steady_clock::now();
    while (!stop.load(std::memory_order_relaxed)) {
      MailEntry* me = &ring[expect % kRing];
      const uint64_t sv = me->seq;
      if ((sv >> 8) != expect) {
        // idle: account completed copies off the critical path (the slot
        // about to be reused first), so issuing an upload never waits on it
        harvest_some();
        // idle: feed the copy engine a speculative chunk when nothing else
        // occupies it (event queries at most every 2 us)
        if (spec_up && (sjob[0].live || sjob[1].live)) {
          const auto now = std::chrono::steady_clock::now();
          if (now - t_poll > std::chrono::microseconds(2)) {
            t_poll = now;
            if (dem_inflight && cudaEventQuery(ev_dem) == cudaSuccess) dem_inflight = false;
            if (spec_inflight && cudaEventQuery(ev_spec) == cudaSuccess) spec_inflight = false;
            if (!dem_inflight && !spec_inflight) {
              // the older job first
              const int b = (sjob[0].live && (!sjob[1].live || sjob[0].gen < sjob[1].gen)) ? 0 : 1;
              issue_spec_chunk((uint32_t)b);
              cudaEventRecord(ev_spec, copy_stream);
              spec_inflight = true;
            }
          }
        }
        // a dedicated poller: the mailbox is the decode loop's critical path
        // (publish -> copy start); yield only after a long idle stretch
        if (++spins > (1u << 20)) std::this_thread::yield();
        else __builtin_ia32_pause();
        continue;
      }
      spins = 0;
      std::atomic_thread_fence(std::memory_order_acquire);
      const uint32_t n = (uint32_t)(sv & 0xff);
      bool uploaded = false;
      for (uint32_t i = 0; i < n; ++i) {
        const MailCmd c = take_cmd(&me->cmd[i], expect);
        if (copier_error) break;
        if (c.kind == 1) {  // a new speculative job (supersedes whatever was left in its buffer)
          SpecJob& j = sjob[c.buf & 1];
          j.gen = c.gen;
          j.chunks = kSpecChunks;
          j.next = 0;
          j.src_off = c.src_off;
          j.dst = c.dst;
          j.bytes = c.bytes;
          j.live = true;
          std::lock_guard<std::mutex> g(io_mu);
          io.spec_jobs += 1;
          continue;
        }
        if (c.kind == 2) {  // promoted: the step needs it now
          SpecJob& j = sjob[c.buf & 1];
          if (j.live && j.gen == c.gen)
            while (j.live) issue_spec_chunk(c.buf & 1);
          std::lock_guard<std::mutex> g(io_mu);
          io.spec_promoted += 1;
          continue;
        }
        if (c.wait_ffn &&
            p_wait32(copy_stream, ffn_ptr, c.wait_ffn, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
          copier_msg = "cuStreamWaitValue32 failed";
          copier_error = 5;
        }
        issue_upload(c, done_ptr);
        uploaded = true;
      }
      if (uploaded && spec_up) {
        cudaEventRecord(ev_dem, copy_stream);
        dem_inflight = true;
      }
      std::atomic_thread_fence(std::memory_order_release);
      *reinterpret_cast<volatile uint64_t*>(ack) = expect;
      ++expect;
    }
  }

  ~moeb_stack() {
    stop = true;
    if (copier.joinable()) copier.join();
    if (stream) cudaStreamSynchronize(stream);
    if (copy_stream) cudaStreamSynchronize(copy_stream);
    for (int i = 0; i < kTk; ++i)
      if (tk_ev[i]) cudaEventDestroy(tk_ev[i]);
    for (int i = 0; i < kEv; ++i) {
      if (ev_a[i]) cudaEventDestroy(ev_a[i]);
      if (ev_b[i]) cudaEventDestroy(ev_b[i]);
    }
    if (pf_copy) cudaStreamSynchronize(pf_copy);
    for (int i = 0; i < 2; ++i) {
      if (pf_up[i]) cudaEventDestroy(pf_up[i]);
      if (pf_free[i]) cudaEventDestroy(pf_free[i]);
    }
    if (pf_copy) cudaStreamDestroy(pf_copy);
    if (ev_spec) cudaEventDestroy(ev_spec);
    if (ev_dem) cudaEventDestroy(ev_dem);
    if (stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (ring) cudaFreeHost(ring);
    if (ack) cudaFreeHost(ack);
    if (own_pool && pool) cudaFreeHost(pool);
    if (registered_pool && pool) cudaHostUnregister(pool);
  }
};

namespace moeb {

static void synth(uint16_t* dst, uint64_t n, uint64_t seed, uint64_t tensor, uint64_t offset, float scale,
                  cudaStream_t s) {
  if (!n) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  synth_kernel<<<grid, 256, 0, s>>>(dst, n, seed, tensor, offset, scale);
  MOEB_CUDA(cudaGetLastError());
}

static void synth_t(uint16_t* dst, uint32_t rows, uint32_t cols, uint64_t seed, uint64_t tensor, float scale,
                    cudaStream_t s) {
  const uint64_t n = (uint64_t)rows * cols;
  if (!n) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  synth_t_kernel<<<grid, 256, 0, s>>>(dst, rows, cols, seed, tensor, scale);
  MOEB_CUDA(cudaGetLastError());
}

static void synth_rows(uint16_t* dst, uint32_t F, uint32_t d, uint64_t seed, uint64_t t0, uint64_t t1, uint64_t t2,
                       float s_in, float s_down, cudaStream_t s) {
  const uint64_t n = 3ull * F * d;
  if (!n) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  synth_rows_kernel<<<grid, 256, 0, s>>>(dst, F, d, seed, t0, t1, t2, s_in, s_down);
  MOEB_CUDA(cudaGetLastError());
}

static void synth_tiled(uint16_t* dst, uint32_t F, uint32_t d, uint64_t seed, uint64_t t0, uint64_t t1, uint64_t t2,
                        float s_in, float s_down, cudaStream_t s) {
  const uint64_t n = 3ull * F * d;
  if (!n) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
  synth_tiled_kernel<<<grid, 256, 0, s>>>(dst, F, d, seed, t0, t1, t2, s_in, s_down);
  MOEB_CUDA(cudaGetLastError());
}

// Tools that serialise kernels inject themselves through these variables
// (ncu/nsys: CUDA_INJECTION64_PATH + NV_COMPUTE_PROFILER_* / NSYS_*;
// compute-sanitizer: its own injection); MOEB_SERIAL=0/1 overrides.
static bool serial_mode_requested() {
  if (const char* v = getenv("MOEB_SERIAL")) return v[0] != '0';
  for (char** e = environ; e && *e; ++e) {
    static const char* kPrefixes[] = {"CUDA_INJECTION64_PATH=", "NV_COMPUTE_PROFILER", "NSYS_", "NV_NSIGHT",
                                      "NV_SANITIZER", "COMPUTE_SANITIZER"};
    for (const char* pre : kPrefixes)
      if (std::strncmp(*e, pre, std::strlen(pre)) == 0) return true;
  }
  return false;
}

static float fan_scale(uint32_t fan_in) { return (float)std::sqrt(3.0 / (double)fan_in); }

// (Re)initialise the decision state and upload the initial residents. The
// layer-step sequence and upload ids stay monotonic across resets: the
// device flags compared against them (copies_done, ffn_done) only grow.
static void reset_state(moeb_stack* S, cudaStream_t s) {
  const uint32_t L = S->L, E = S->E;
  const uint64_t eb = S->expert_elems * 2;
  std::vector<LayerState> ls;
  init_layers(S->dcfg, S->cfg.init_fill, S->cfg.seed, ls);
  EngineState prev{};
  MOEB_CUDA(cudaMemcpyAsync(&prev, S->st.p, sizeof prev, cudaMemcpyDeviceToHost, s));
  MOEB_CUDA(cudaStreamSynchronize(s));
  EngineState st{};
  rng_seed(st.rng, derive_seed(S->cfg.seed, 0x94ed1c70ULL));  // pipeline.cpp:62
  st.seq = prev.seq;
  st.next_copy = prev.next_copy;
  st.sp_gen_next = prev.sp_gen_next;  // spec_done only grows
  st.ack_cache = prev.ack_cache;
  st.prof[14] = ~0ull;  // running minimum of CTA start times (phase profiling)
  S->hist.zero(s);
  MOEB_CUDA(cudaMemcpyAsync(S->st.p, &st, sizeof st, cudaMemcpyHostToDevice, s));
  MOEB_CUDA(cudaMemcpyAsync(S->layers.p, ls.data(), L * sizeof(LayerState), cudaMemcpyHostToDevice, s));
  for (uint32_t l = 0; l < L; ++l)
    for (uint32_t e = 0; e < E; ++e)
      if (ls[l].slot_of[e] >= 0)
        MOEB_CUDA(cudaMemcpyAsync(S->slots.p + ((size_t)l * S->slots_alloc + ls[l].slot_of[e]) * S->expert_elems,
                                  reinterpret_cast<char*>(S->pool) + ((uint64_t)l * E + e) * eb, eb,
                                  cudaMemcpyHostToDevice, s));
  MOEB_CUDA(cudaStreamSynchronize(s));
}

static void build_stack(moeb_stack* S, const moeb_config& cfg, const moeb_model& m, const void* weights_host,
                        int device) {
  validate(cfg);
  if (m.d_model == 0 || m.d_model % 256) throw Error(1, "model: d_model must be a positive multiple of 256");
  if (m.ffn == 0 || m.ffn % 8) throw Error(1, "model: ffn must be a positive multiple of 8");
  if (m.shared_ffn % 8) throw Error(1, "model: shared_ffn must be a multiple of 8");
  if ((size_t)cfg.batch * m.d_model * 2 > 160 * 1024) throw Error(1, "model: batch * d_model too large for the FFN tile");
  if (cfg.slots > (uint32_t)kMaxSlots) throw Error(1, "device engine: slots_per_layer must be <= 64");
  S->cfg = cfg;
  S->model = m;
  S->dcfg = make_dev_cfg(cfg);
  S->device = device;
  S->L = cfg.num_layers;
  S->E = cfg.experts;
  S->B = cfg.batch;
  S->d = m.d_model;
  S->F = m.ffn;
  S->S = m.shared_ffn;
  S->slots_alloc = std::max<uint32_t>(std::min(cfg.slots, cfg.experts), 1);
  S->expert_elems = 3ull * m.ffn * m.d_model;
  S->n_stage = std::max<uint32_t>(1, std::min<uint32_t>(cfg.experts, cfg.batch * cfg.top_k));
  MOEB_CUDA(cudaSetDevice(device));
  MOEB_CUDA(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
  MOEB_CUDA(cudaStreamCreateWithFlags(&S->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < moeb_stack::kEv; ++i) {
    MOEB_CUDA(cudaEventCreate(&S->ev_a[i]));
    MOEB_CUDA(cudaEventCreate(&S->ev_b[i]));
  }
  if (m.flags & MOEB_MODEL_TIME_KERNELS) {
    S->timing = true;
    for (int i = 0; i < moeb_stack::kTk; ++i) MOEB_CUDA(cudaEventCreate(&S->tk_ev[i]));
  }
  load_stream_memops();
  const cudaStream_t s = S->stream;
  const uint32_t L = S->L, E = S->E, B = S->B, d = S->d, F = S->F, Sh = S->S;
  const uint64_t seed = m.weight_seed;
  // batch 1: split-K FFN over row-interleaved experts ([F][3][d])
  int n_sm = 0;
  MOEB_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device));
  // (the split-K FFN's final sum gathers <= 16 outputs per CTA: d <= 16 (SMs - 1))
  S->splitk = B == 1 && d <= 2048 && d <= 16u * (uint32_t)(n_sm - 1) && getenv("MOEB_NO_SPLITK") == nullptr;
  if (const char* ur = getenv("MOEB_SK_UNIT")) S->unit_rows = (uint32_t)atoi(ur);
  if (const char* fd = getenv("MOEB_FFN_DBG")) S->ffn_dbg = (uint32_t)atoi(fd);  // microbenchmark knob
  S->sk_shared_prefetch = getenv("MOEB_NO_SHARED_PREFETCH") == nullptr;
  // batch 2..32: tensor-core FFN over UMMA-tiled experts, when the shapes
  // tile (ffn, shared_ffn multiples of 128) and the pool is ours to lay out
  // (or a caller pool declares the tiled layout). MOEB_NO_UMMA=1 selects the
  // CUDA-core FFN over HF layouts.
  const bool own_layout = !weights_host || (m.flags & MOEB_MODEL_FILL_POOL);
  S->umma = B >= 2 && B <= 32 && F % 128 == 0 && Sh % 128 == 0 && d / 64 <= 148 &&
            (own_layout || (m.flags & MOEB_MODEL_TILED)) && getenv("MOEB_NO_UMMA") == nullptr;
  if (weights_host && !own_layout && S->layout_flags() != (m.flags & (MOEB_MODEL_DOWN_T | MOEB_MODEL_TILED)))
    throw Error(1, S->splitk ? "model: a batch-1 stack needs a row-interleaved host pool (MOEB_MODEL_DOWN_T)"
                             : "model: this stack needs a host pool in the [gate][up][down] layout (no MOEB_MODEL_DOWN_T)");
  // resident (HBM) weights: router, shared expert, shared gate
  S->gate_w.alloc((size_t)L * E * d);
  for (uint32_t l = 0; l < L; ++l) synth(S->gate_w.p + (size_t)l * E * d, (uint64_t)E * d, seed, tid_router(l), 0, fan_scale(d), s);
  if (Sh) {
    S->shared_w.alloc((size_t)L * 3 * Sh * d);
    for (uint32_t l = 0; l < L; ++l) {
      uint16_t* base = S->shared_w.p + (size_t)l * 3 * Sh * d;
      if (S->splitk) {
        synth_rows(base, Sh, d, seed, tid_shared(l, 0), tid_shared(l, 1), tid_shared(l, 2), fan_scale(d), fan_scale(Sh), s);
      } else if (S->umma) {
        synth_tiled(base, Sh, d, seed, tid_shared(l, 0), tid_shared(l, 1), tid_shared(l, 2), fan_scale(d), fan_scale(Sh), s);
      } else {
        synth(base, (uint64_t)Sh * d, seed, tid_shared(l, 0), 0, fan_scale(d), s);
        synth(base + (size_t)Sh * d, (uint64_t)Sh * d, seed, tid_shared(l, 1), 0, fan_scale(d), s);
        synth(base + 2 * (size_t)Sh * d, (uint64_t)Sh * d, seed, tid_shared(l, 2), 0, fan_scale(Sh), s);
      }
    }
  }
  if (m.shared_gate) {
    S->sgate_w.alloc((size_t)L * d);
    for (uint32_t l = 0; l < L; ++l) synth(S->sgate_w.p + (size_t)l * d, d, seed, tid_shared_gate(l), 0, fan_scale(d), s);
  }
  // pinned host pool of every routed expert
  const uint64_t eb = S->expert_elems * 2;
  const uint64_t pool_bytes = (uint64_t)L * E * eb;
  const bool fill = weights_host && (m.flags & MOEB_MODEL_FILL_POOL);
  if (weights_host) {
    S->pool = const_cast<uint16_t*>(static_cast<const uint16_t*>(weights_host));
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, weights_host) != cudaSuccess || pa.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      MOEB_CUDA(cudaHostRegister(S->pool, pool_bytes, cudaHostRegisterPortable));
      S->registered_pool = true;
    }
  } else {
    MOEB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&S->pool), pool_bytes, cudaHostAllocPortable));
    S->own_pool = true;
  }
  if (!weights_host || fill) {
    // generate on the device, expert by expert, then D2H into the pool
    DevBuf<uint16_t> tmp(2 * S->expert_elems);
    for (uint64_t i = 0; i < (uint64_t)L * E; ++i) {
      const uint32_t l = (uint32_t)(i / E), e = (uint32_t)(i % E);
      uint16_t* buf = tmp.p + (i & 1) * S->expert_elems;
      if (S->splitk) {
        synth_rows(buf, F, d, seed, tid_expert(l, e, 0), tid_expert(l, e, 1), tid_expert(l, e, 2), fan_scale(d),
                   fan_scale(F), s);
      } else if (S->umma) {
        synth_tiled(buf, F, d, seed, tid_expert(l, e, 0), tid_expert(l, e, 1), tid_expert(l, e, 2), fan_scale(d),
                    fan_scale(F), s);
      } else {
        synth(buf, (uint64_t)F * d, seed, tid_expert(l, e, 0), 0, fan_scale(d), s);
        synth(buf + (size_t)F * d, (uint64_t)F * d, seed, tid_expert(l, e, 1), 0, fan_scale(d), s);
        synth(buf + 2 * (size_t)F * d, (uint64_t)F * d, seed, tid_expert(l, e, 2), 0, fan_scale(F), s);
      }
      MOEB_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(S->pool) + i * eb, buf, eb, cudaMemcpyDeviceToHost, s));
    }
    MOEB_CUDA(cudaStreamSynchronize(s));
  }
  // expert cache slots + staging
  S->slots.alloc((size_t)L * S->slots_alloc * S->expert_elems);
  S->staging.alloc((size_t)S->n_stage * S->expert_elems);
  S->hidden.alloc(2ull * B * d);
  S->u.alloc((size_t)B * d);
  S->logits.alloc((size_t)B * (E + 1));
  const uint32_t Fmax = std::max(F, Sh);
  S->h.alloc((size_t)kMaxItems * kMaxB * Fmax);
  S->y_layers.alloc((size_t)L * B * d);
  S->y_layers.zero(s);
  // decision engine state + initial residency
  S->st.alloc(1);
  S->layers.alloc(L);
  S->hist.alloc((size_t)L * cfg.window * E);
  EngineState st0{};
  MOEB_CUDA(cudaMemcpyAsync(S->st.p, &st0, sizeof st0, cudaMemcpyHostToDevice, s));
  reset_state(S, s);
  S->plan.alloc(1);
  // speculative FFN start (batch 1, combine weights known at classification)
  // (the batched tcgen05 FFN takes the combine weights from the final plan,
  // so it also runs with renormalised weights)
  S->spec = ((B == 1 && !m.renormalize) || S->umma) && getenv("MOEB_NO_SPEC") == nullptr;
  if (S->spec) {
    S->spec_plan.alloc(1);
    S->spec_flag.alloc(3);  // [0] speculative plan published, [1] final plan published, [2] shared expert released
    S->spec_flag.zero(s);
  }
  if (getenv("MOEB_FFN_TSTAMP")) {
    S->ffn_ts.alloc(8 * (size_t)n_sm);  // [CTA][8]: the split-K grid is at most one CTA per SM
    S->ffn_ts.zero(s);
  }
  S->ffn_ctr.alloc(kFfnCtrWords);
  S->ffn_ctr.zero(s);
  S->copies_done.alloc(1);
  S->copies_done.zero(s);
  S->ffn_done.alloc(1);
  S->ffn_done.zero(s);
  if (m.flags & MOEB_MODEL_TRACE_TIMELINE) {
    S->timeline.alloc(16384 * kTlWords);
    S->timeline.zero(s);
  }
  if (m.flags & MOEB_MODEL_LOG_STEPS) {
    S->rec_cap = 16384;
    S->recs.alloc(S->rec_cap);
    S->toks.alloc(S->rec_cap * B);
    S->scores_log.alloc(S->rec_cap * B * E);
  }
  S->predictor = (m.flags & MOEB_MODEL_PREDICTOR) != 0;
  if (S->predictor) {
    if (!S->splitk && !S->umma)
      throw Error(1, "model: the predictor needs the split-K (batch 1, d_model <= 2048) or the tensor-core "
                     "(batch 2..32, ffn and shared_ffn multiples of 128) FFN");
    S->xpred.alloc((size_t)B * d);
    S->xpred.zero(s);
    S->plogits.alloc((size_t)B * (E + 1));
    S->plogits.zero(s);
    if (S->rec_cap) {
      S->pred_log.alloc(S->rec_cap * B * E);
      MOEB_CUDA(cudaMemsetAsync(S->pred_log.p, 0xff, S->rec_cap * B * E * sizeof(float), s));  // NaN: no prediction
    }
  }
  MOEB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&S->ring), sizeof(MailEntry) * kRing, cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(S->ring, 0, sizeof(MailEntry) * kRing);
  MOEB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&S->ack), 64, cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(S->ack, 0, 64);
  // kernel resources: FFN launch shape (ring stages, h staging, accumulators)
  int sms = 0;
  MOEB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  if (S->umma) {
    S->um = umma_launch_config(B, d, 1 + std::min(E, B * cfg.top_k));
    S->xt.alloc((size_t)(d / 64) * S->um.Nx * 64);
    S->xt.zero(s);  // token rows >= B stay zero
    const uint64_t n_exp = std::min<uint64_t>(E, (uint64_t)B * cfg.top_k);
    const uint64_t tiles = Sh / 128 + n_exp * (F / 128);
    const uint64_t parts = (Sh / 128 + S->um.dn_st - 1) / S->um.dn_st + n_exp * ((F / 128 + S->um.dn_st - 1) / S->um.dn_st);
    S->part.alloc(parts * B * d);
    S->gpart.alloc(tiles * S->um.KS * 2 * S->um.Nx * 128);
    S->gcnt.alloc(tiles);
    S->gcnt.zero(s);
  }
  S->ffn = S->splitk ? ffn_splitk_config(d, E, cfg.top_k, 8, getenv("MOEB_DYNAMIC_ROWS") == nullptr)
                     : ffn_launch_config(B, d, F, Sh, E, cfg.top_k, S->spec ? sms - 1 : sms);
  if (S->umma) {
    S->ffn.fn = reinterpret_cast<void (*)(FfnTArgs)>(ffn_umma_kernel);
    S->ffn.threads = kUmThreads;
    S->ffn.stages = S->um.stages;
    S->ffn.stage_bytes = S->um.stage_bytes;
    S->ffn.smem = S->um.smem;
  }
  if (S->ffn.stages < 2) throw Error(1, "model: batch * d_model too large for the FFN pipeline");
  S->ticket.alloc(1);
  S->ticket.zero(s);
  MOEB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&S->ring_dev), S->ring, 0));
  MOEB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&S->ack_dev), S->ack, 0));
  S->gd_smem = std::max<size_t>((size_t)B * d * 2, sizeof(DecideKSmem));
  MOEB_CUDA(cudaFuncSetAttribute(gate_decide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->gd_smem));
  // one shared-memory carveout for both per-layer kernels: no L1/smem
  // reconfiguration drain between them
  MOEB_CUDA(cudaFuncSetAttribute(gate_decide_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  MOEB_CUDA(cudaFuncSetAttribute(S->ffn.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->ffn.smem));
  MOEB_CUDA(cudaFuncSetAttribute(S->ffn.fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int occ = 0;
  MOEB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, S->ffn.fn, S->ffn.threads, S->ffn.smem));
  if (occ < 1) throw Error(5, "ffn kernel does not fit on an SM");
  // one persistent CTA per SM (the grid counters need co-residency); with
  // the speculative start the FFN runs beside the deciding CTA, so one SM
  // is left to it
  S->ffn_grid = S->spec ? sms - 1 : sms;
  S->serial = S->serial_at_create = serial_mode_requested();
  // speculative uploads (opt-in, MOEB_SPEC_UPLOAD=1): the split-K (batch-1)
  // path with stage Pre and a capped cache; not in serial (profiler) mode.
  // Measured on the bench workload: 9.91 vs 7.86 ms/token without — half the
  // guesses are wrong, chunked copies run at ~44 vs ~53 GB/s, a wrong guess
  // delays the next real upload by a chunk, and a right one costs a buffer ->
  // slot copy in the FFN epilogue. Kept as an experiment.
  const char* spv = getenv("MOEB_SPEC_UPLOAD");
  S->spec_up = spv && spv[0] == '1' && S->splitk && cfg.pre && cfg.slots < cfg.experts && !S->serial &&
               !S->predictor;
  if (S->spec_up) {
    S->specbuf.alloc(2 * S->expert_elems);
    S->spec_done.alloc(2);
    S->spec_done.zero(s);
    MOEB_CUDA(cudaEventCreateWithFlags(&S->ev_spec, cudaEventDisableTiming));
    MOEB_CUDA(cudaEventCreateWithFlags(&S->ev_dem, cudaEventDisableTiming));
  }
  // upload destinations travel as 48-bit words (WireCmd)
  for (const void* q : {static_cast<const void*>(S->slots.p + S->slots.n), static_cast<const void*>(S->staging.p + S->staging.n),
                        static_cast<const void*>(S->specbuf.p + S->specbuf.n)})
    if ((uint64_t)q >> 48) throw Error(5, "device addresses above 2^48 are not supported by the upload mailbox");
  if (S->serial && !getenv("MOEB_SERIAL"))
    fprintf(stderr, "moeb: profiler detected, serial pipeline mode (set MOEB_SERIAL=0 to override)\n");
  MOEB_CUDA(cudaStreamSynchronize(s));
  S->copier = std::thread([S] { S->copy_loop(); });
}

// Programmatic dependent launch: the next per-layer kernel is scheduled while
// the current one drains (each kernel opens with griddepcontrol.wait, so
// data dependences are unchanged), hiding the grid launch latency between
// the gate+decide and FFN kernels of every layer. Measured on B200 (device
// timeline, DSV2-Lite B=1): decide end -> FFN start 4.4 -> 2.0 us, FFN end ->
// next decide 6.5 -> 4.8 us. MOEB_NO_PDL=1 turns it off.
static const bool kUsePdl = getenv("MOEB_NO_PDL") == nullptr;

template <class Args>
static void launch_pdl(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args* args,
                       bool pdl = kUsePdl) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* kargs[] = {args};
  MOEB_CUDA(cudaLaunchKernelExC(&cfg, fn, kargs));
}

// Serial mode, after layer-step `seq`'s decide kernel was launched: wait for
// it, read the upload commands it published (mailbox entries A = demand loads
// and BA streams of this step, B = prefetches for later steps) and make the
// compute stream wait for every upload the coming FFN may read. Upload ids
// grow in publication order and the copy stream is FIFO, so one
// copies_done >= id wait covers them; entry B's prefetches (which themselves
// wait for this step's FFN) are only owed to later steps.
static void serial_wait_uploads(moeb_stack* S, cudaStream_t s, uint64_t seq) {
  MOEB_CUDA(cudaStreamSynchronize(s));
  // the copy thread must have ISSUED entry A's copies before the FFN launch:
  // a profiler holds every API call (the copy thread's too) while it
  // measures a kernel, and the FFN depends on those copies
  const auto t0 = std::chrono::steady_clock::now();
  while (*reinterpret_cast<volatile uint64_t*>(S->ack) < 2 * seq - 1) {
    if (S->copier_error) throw Error(5, S->copier_msg);
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20))
      throw Error(5, "serial mode: the copy thread did not take the step's upload commands");
    std::this_thread::yield();
  }
  const MailEntry* ea = &S->ring[(2 * seq - 1) % kRing];
  // entry B of this step, or (predictor mode) of the previous one, which this
  // step's kernel published before entry A
  const uint64_t bseq = S->predictor ? 2 * seq - 2 : 2 * seq;
  const MailEntry* eb = &S->ring[bseq % kRing];
  const uint64_t va = ea->seq, vb = bseq ? eb->seq : 0;
  if ((va >> 8) != 2 * seq - 1 || (bseq && (vb >> 8) != bseq))
    throw Error(5, "serial mode: the decide kernel did not publish its upload commands");
  // the upload id of an entry's last command (its words carry the entry's
  // tag once they have arrived: WireCmd)
  auto last_id = [&](const MailEntry* e, uint64_t mseq, uint64_t sv) -> uint32_t {
    const volatile uint64_t* w3 = &e->cmd[(sv & 0xff) - 1].w[3];
    const auto t1 = std::chrono::steady_clock::now();
    while ((*w3 >> 48) != (mseq & 0xffff))
      if (std::chrono::steady_clock::now() - t1 > std::chrono::seconds(5))
        throw Error(5, "serial mode: mailbox command words did not arrive");
    return (uint32_t)*w3;
  };
  if (S->predictor && (vb & 0xff)) S->serial_need = std::max(S->serial_need, last_id(eb, bseq, vb));
  if (va & 0xff) S->serial_need = std::max(S->serial_need, last_id(ea, 2 * seq - 1, va));
  if (S->serial_need &&
      p_wait32(s, (CUdeviceptr)S->copies_done.p, S->serial_need, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    throw Error(5, "serial mode: cuStreamWaitValue32 failed");
  if (!S->predictor && (vb & 0xff)) S->serial_need = std::max(S->serial_need, last_id(eb, bseq, vb));
}

// The persistent FFN grids assume every CTA is co-resident (grid barriers,
// one CTA per SM). Two stacks stepping on one GPU at the same time could each
// end up partly resident, so the steps of all stacks of a device are ordered:
// a stack's step waits (on the device, through an event) for the last step
// any other stack of that device enqueued.
struct DeviceOrder {
  std::mutex mu;
  cudaEvent_t ev = nullptr;
  const moeb_stack* owner = nullptr;
};
static DeviceOrder& device_order(int dev) {
  static DeviceOrder orders[64];
  return orders[dev & 63];
}

static void step_stack_locked(moeb_stack* S, const void* x, void* y, uint32_t B, cudaStream_t s);

static void step_stack(moeb_stack* S, const void* x, void* y, uint32_t B, cudaStream_t user) {
  if (B != S->B) throw Error(1, "step: batch must equal the configured batch_size");
  if (S->copier_error) throw Error(5, S->copier_msg);
  if (S->cfg.pre && !S->trace.p && !S->predictor)
    throw Error(1, "stage Pre needs a logits trace (moeb_set_logits_trace) or the predictor (MOEB_MODEL_PREDICTOR)");
  cudaStream_t s = user ? user : S->stream;
  MOEB_CUDA(cudaSetDevice(S->device));
  DeviceOrder& o = device_order(S->device);
  std::lock_guard<std::mutex> lk(o.mu);
  if (!o.ev) MOEB_CUDA(cudaEventCreateWithFlags(&o.ev, cudaEventDisableTiming));
  if (o.owner && o.owner != S) MOEB_CUDA(cudaStreamWaitEvent(s, o.ev, 0));
  step_stack_locked(S, x, y, B, s);
  MOEB_CUDA(cudaEventRecord(o.ev, s));
  o.owner = S;
}

static void step_stack_locked(moeb_stack* S, const void* x, void* y, uint32_t B, cudaStream_t s) {
  const uint32_t L = S->L, E = S->E, d = S->d;
  MOEB_CUDA(cudaMemcpyAsync(S->hidden.p, x, (size_t)B * d * 2, cudaMemcpyDeviceToDevice, s));
  int cur = 0;
  for (uint32_t l = 0; l < L; ++l) {
    GateDecideArgs ga{};
    GateArgs& g = ga.g;
    g.x = S->hidden.p + (size_t)cur * B * d;
    g.wg = S->gate_w.p + (size_t)l * E * d;
    g.wsg = S->model.shared_gate ? S->sgate_w.p + (size_t)l * d : nullptr;
    g.u = S->u.p;
    g.ut = S->umma ? S->xt.p : nullptr;
    g.ut_rows = S->um.Nx;
    g.logits = S->logits.p;
    g.x_pred = S->predictor ? S->xpred.p : nullptr;
    g.plogits = S->predictor ? S->plogits.p : nullptr;
    g.B = B;
    g.d = d;
    g.E = E;
    const uint32_t rows = E + (g.wsg ? 1 : 0);
    DecideArgs& a = ga.d;
    a.cfg = S->dcfg;
    a.st = S->st.p;
    a.layers = S->layers.p;
    a.hist = S->hist.p;
    a.layer = l;
    a.logits = S->logits.p;
    a.trace = S->trace.p;
    a.trace_steps = S->trace_steps;
    a.total_iters = S->total_iters;
    a.shared_gate = S->model.shared_gate;
    a.renormalize = S->model.renormalize;
    a.routed_scale = S->model.routed_scale;
    a.shared_w = S->S ? S->shared_w.p + (size_t)l * 3 * S->S * d : nullptr;
    a.S = S->S;
    a.F = S->F;
    a.d = d;
    a.slots_alloc = S->slots_alloc;
    a.slots = S->slots.p;
    a.staging = S->staging.p;
    a.n_stage = S->n_stage;
    a.expert_elems = S->expert_elems;
    a.plan = S->plan.p;
    a.spec_plan = S->spec ? S->spec_plan.p : nullptr;
    a.spec_flag = S->spec_flag.p;
    a.ffn_ctr = S->ffn_ctr.p;
    a.copies_done = S->copies_done.p;
    a.ring = S->ring_dev;
    a.host_ack = S->ack_dev;
    a.scores_log = S->scores_log.p;
    a.recs = S->recs.p;
    a.toks = S->toks.p;
    a.rec_cap = S->rec_cap;
    a.it = S->host_it;
    a.seq = ++S->host_seq;
    a.tl = S->timeline.p ? S->timeline.p + ((a.seq - 1) % 16384) * kTlWords : nullptr;
    a.predictor = S->predictor ? 1u : 0u;
    a.shared_first = (S->spec && S->splitk && S->S && getenv("MOEB_NO_SHARED_FIRST") == nullptr) ? 1u : 0u;
    a.spec_up = S->spec_up ? 1u : 0u;
    a.specbuf = S->specbuf.p;
    a.plogits = S->plogits.p;
    a.pred_log = S->pred_log.p;
    ga.ticket = S->ticket.p;
    if (S->timing) S->tick(s);
    launch_pdl(reinterpret_cast<const void*>(gate_decide_kernel), dim3(1 + (rows + 1) / 2), dim3(kGdThreads),
               S->gd_smem, s, &ga, kUsePdl && !S->serial);
    MOEB_CUDA(cudaGetLastError());
    if (S->serial) serial_wait_uploads(S, s, a.seq);
    if (S->timing) S->tick(s);

    FfnTArgs f{};
    f.plan = S->plan.p;
    f.u = S->u.p;
    f.x_in = S->hidden.p + (size_t)cur * B * d;
    f.x_out = S->hidden.p + (size_t)(cur ^ 1) * B * d;
    f.y_out = S->y_layers.p + (size_t)l * B * d;
    f.x_pred = S->predictor ? S->xpred.p : nullptr;
    f.h = S->h.p;
    f.ctr = S->ffn_ctr.p;
    f.copies_done = S->copies_done.p;
    f.ffn_done = S->ffn_done.p;
    f.B = B;
    f.d = d;
    f.Fmax = std::max(S->F, S->S);
    f.stages = S->ffn.stages;
    f.stage_bytes = S->ffn.stage_bytes;
    f.hbuf_bytes = S->ffn.hbuf_bytes;
    f.acc_rows = S->ffn.acc_rows;
    f.plan_smem = S->ffn.plan_smem;
    f.tl = a.tl;
    f.tstamp = S->splitk ? S->ffn_ts.p : nullptr;
    f.spec_plan = a.spec_plan;
    f.spec_flag = S->spec_flag.p;
    f.shared_first = a.shared_first;
    f.shared_w = S->sk_shared_prefetch ? a.shared_w : nullptr;
    f.shared_F = a.S;
    f.spec_done = S->spec_done.p;
    f.seq = (uint32_t)a.seq;
    f.unit_rows = S->unit_rows;
    // rows are dealt round-robin to the CTAs (fixed partial sums, no counter
    // atomics; measured faster than the grid-dynamic grab on B200, 50 vs 53 us
    // per all-resident layer). MOEB_DYNAMIC_ROWS=1 selects the dynamic grab.
    f.deterministic = getenv("MOEB_DYNAMIC_ROWS") ? 0u : 1u;
    f.dbg = S->ffn_dbg;
    f.x_smem = S->ffn.x_smem;
    if (S->umma) {
      UmArgs ua{};
      ua.f = f;
      ua.xt = S->xt.p;
      ua.part = S->part.p;
      ua.Nx = S->um.Nx;
      ua.Bp = S->um.Bp;
      ua.stages = S->um.stages;
      ua.stage_bytes = S->um.stage_bytes;
      ua.gpart = S->gpart.p;
      ua.gcnt = S->gcnt.p;
      ua.KS = S->um.KS;
      ua.dn_st = S->um.dn_st;
      launch_pdl(reinterpret_cast<const void*>(S->ffn.fn), dim3(S->ffn_grid), dim3(S->ffn.threads), S->ffn.smem, s,
                 &ua, kUsePdl && !S->serial);
    } else {
      launch_pdl(reinterpret_cast<const void*>(S->ffn.fn), dim3(S->ffn_grid), dim3(S->ffn.threads), S->ffn.smem, s,
                 &f, kUsePdl && !S->serial);
    }
    S->n_launch_layers += 1;
    MOEB_CUDA(cudaGetLastError());
    if (S->timing) S->tick(s);
    cur ^= 1;
  }
  MOEB_CUDA(cudaMemcpyAsync(y, S->hidden.p + (size_t)cur * B * d, (size_t)B * d * 2, cudaMemcpyDeviceToDevice, s));
  S->host_it += 1;
  std::lock_guard<std::mutex> g(S->io_mu);
  S->io.steps += 1;
}

// Uploads the last decode steps decided (prefetches into cache slots) may
// still be with the copy thread after the compute stream is idle: wait until
// it has taken every published mailbox entry, then for its copy stream.
// Callers have synchronised the stream the steps ran on.
static void drain_uploads(moeb_stack* S) {
  const uint64_t want = S->predictor ? (S->host_seq ? 2 * S->host_seq - 1 : 0) : 2 * S->host_seq;
  const auto t0 = std::chrono::steady_clock::now();
  while (*reinterpret_cast<volatile uint64_t*>(S->ack) < want) {
    if (S->copier_error) throw Error(5, S->copier_msg);
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20))
      throw Error(5, "the copy thread did not take the decode steps' upload commands");
    std::this_thread::yield();
  }
  MOEB_CUDA(cudaStreamSynchronize(S->copy_stream));
}

// ---------------------------------------------------------------- prefill
// N prompt tokens through all L layers (prefill.cuh). Plain top-k routing
// (no substitution, no cache admission: the decode state is untouched —
// PAPER.md:358-362), every selected expert computed on the tensor cores.
// Experts not resident in the capped cache are uploaded into a per-layer
// staging area from the pinned pool, layer l+1's while layer l computes (the
// paper's prefill pipeline); all of them, since prefill activation is dense
// (PAPER.md:770-774).
static void prefill_alloc(moeb_stack* S, uint32_t N) {
  const uint32_t E = S->E, k = S->cfg.top_k, d = S->d, Fmax = std::max(S->F, S->S);
  const cudaStream_t s = S->stream;
  if (N > S->pf_cap) {
    const uint32_t R = ((N + 15) & ~15u) + N * k + 16 * E;
    const uint32_t tiles = (N + kPfNt - 1) / kPfNt + (N * k + kPfNt - 1) / kPfNt + E;
    S->pf_u.alloc((size_t)N * d);
    S->pf_hid.alloc((size_t)2 * N * d);
    S->pf_logits.alloc((size_t)N * (E + 1));
    S->pf_scores.alloc((size_t)N * E);
    S->pf_wts.alloc((size_t)N * k);
    S->pf_sel.alloc((size_t)N * k);
    S->pf_entry.alloc((size_t)N * k);
    S->pf_slot_w.alloc(R);
    S->pf_out.alloc((size_t)R * d);
    S->pf_xg.alloc((size_t)R * d * 2);
    S->pf_hg.alloc((size_t)R * Fmax * 4);
    S->pf_hg.zero(s);
    S->pf_ctr.alloc(2 + tiles);
    S->pf_items.alloc(kMaxItems);
    S->pf_hdr.alloc(1);
    if (!S->pf_cnt.p) {
      S->pf_cnt.alloc(kMaxE + 1);  // histogram + the top-k kernel's ticket
      S->pf_cnt.zero(s);
      S->pf_cursor.alloc(kMaxE);
    }
    S->pf_cap = N;
    S->pf_R = R;
    S->pf_tiles = tiles;
  }
  if (!S->pf_copy) {
    MOEB_CUDA(cudaStreamCreateWithFlags(&S->pf_copy, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      MOEB_CUDA(cudaEventCreateWithFlags(&S->pf_up[i], cudaEventDisableTiming));
      MOEB_CUDA(cudaEventCreateWithFlags(&S->pf_free[i], cudaEventDisableTiming));
    }
    MOEB_CUDA(cudaFuncSetAttribute(pf_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(kPfStages * kPfStageBytes + 1024)));
    MOEB_CUDA(cudaFuncSetAttribute(pf_router_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(kPfRouterTok * (d + 8) * 2)));
  }
  if (S->rec_cap && N > S->pf_log_n) {
    const uint32_t L = S->L;
    S->pf_log_x.alloc((size_t)L * N * d);
    S->pf_log_scores.alloc((size_t)L * N * E);
    S->pf_log_y.alloc((size_t)L * N * d);
    S->pf_log_sel.alloc((size_t)L * N * k);
    S->pf_log_n = N;
  }
}

static uint64_t prefill_stack(moeb_stack* S, const void* x, void* y, uint32_t N, cudaStream_t s) {
  const uint32_t L = S->L, E = S->E, k = S->cfg.top_k, d = S->d, F = S->F, Sh = S->S;
  if (!S->umma && !(S->splitk && F % 128 == 0 && Sh % 128 == 0))
    throw Error(1, "prefill needs the UMMA-tiled expert layout (max_batch 2..32) or the row-interleaved one "
                   "(batch 1, d_model <= 2048), with ffn and shared_ffn multiples of 128");
  if (N == 0) throw Error(1, "prefill: no tokens");
  if (k > kPfMaxK) throw Error(1, "prefill: top_k > 16");
  prefill_alloc(S, N);
  // the cache residency (which experts to upload): read once, unless every
  // expert fits the cache and the initial fill put them all there (then
  // nothing is ever evicted: no host sync)
  const uint64_t all = E == 64 ? ~0ull : ((1ull << E) - 1);
  std::vector<LayerState> ls(L);
  if (S->cfg.slots >= E && S->cfg.init_fill != 2) {
    for (uint32_t l = 0; l < L; ++l) ls[l].mask = all;
  } else {
    MOEB_CUDA(cudaStreamSynchronize(s));
    // every resident slot must hold its expert before the GEMM reads it
    drain_uploads(S);
    MOEB_CUDA(cudaMemcpy(ls.data(), S->layers.p, sizeof(LayerState) * L, cudaMemcpyDeviceToHost));
  }
  const uint64_t eb = S->expert_elems * 2;
  bool any_up = false;
  for (uint32_t l = 0; l < L; ++l)
    if (ls[l].mask != all) any_up = true;
  if (any_up && !S->pf_stage.p) S->pf_stage.alloc(2 * (size_t)E * S->expert_elems);
  // batch-1 stacks: experts are row-interleaved; every layer is re-tiled
  // into one buffer (routed experts by id, then the shared expert)
  const bool retile = !S->umma;
  if (retile && !S->pf_tiled.p) S->pf_tiled.alloc((size_t)E * S->expert_elems + (size_t)3 * Sh * d);
  uint64_t h2d = 0;
  std::vector<char> up(L, 0);
  auto upload = [&](uint32_t l) {
    unsigned char* dst = reinterpret_cast<unsigned char*>(S->pf_stage.p) + (size_t)(l % 2) * E * eb;
    const unsigned char* src = reinterpret_cast<const unsigned char*>(S->pool) + (size_t)l * E * eb;
    for (uint32_t e = 0; e < E;) {
      if ((ls[l].mask >> e) & 1ull) {
        ++e;
        continue;
      }
      uint32_t e1 = e;
      // a run of non-resident experts: one copy from the host pool (per expert
      // from a device tier, moeb_set_expert_sources)
      while (e1 < E && !((ls[l].mask >> e1) & 1ull) && (e1 == e || S->src_tab.empty())) ++e1;
      MOEB_CUDA(cudaMemcpyAsync(dst + (size_t)e * eb, S->src_tab.empty() ? static_cast<const void*>(src + (size_t)e * eb)
                                                                         : S->upload_src(((uint64_t)l * E + e) * eb),
                                (size_t)(e1 - e) * eb, cudaMemcpyDefault, S->pf_copy));
      h2d += (uint64_t)(e1 - e) * eb;
      up[l] = 1;
      e = e1;
    }
    MOEB_CUDA(cudaEventRecord(S->pf_up[l % 2], S->pf_copy));
  };
  int n_sm = 0;
  MOEB_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, S->device));
  const size_t r_smem = (size_t)kPfRouterTok * (d + 8) * 2;
  const bool log = S->rec_cap != 0;
  if (any_up) upload(0);
  for (uint32_t l = 0; l < L; ++l) {
    if (any_up && l + 1 < L) {
      if (l >= 1) MOEB_CUDA(cudaStreamWaitEvent(S->pf_copy, S->pf_free[(l + 1) % 2], 0));
      upload(l + 1);
    }
    if (up[l]) MOEB_CUDA(cudaStreamWaitEvent(s, S->pf_up[l % 2], 0));
    const uint16_t* xin = l == 0 ? static_cast<const uint16_t*>(x) : S->pf_hid.p + (size_t)((l - 1) % 2) * N * d;
    uint16_t* xout = l + 1 == L ? static_cast<uint16_t*>(y) : S->pf_hid.p + (size_t)(l % 2) * N * d;
    PfRouterArgs ra{};
    ra.x = xin;
    ra.wg = S->gate_w.p + (size_t)l * E * d;
    ra.wsg = S->model.shared_gate ? S->sgate_w.p + (size_t)l * d : nullptr;
    ra.u = S->pf_u.p;
    ra.xg = Sh ? S->pf_xg.p : nullptr;
    ra.logits = S->pf_logits.p;
    ra.N = N;
    ra.d = d;
    ra.E = E;
    ra.R = S->pf_R;
    launch_pdl(reinterpret_cast<const void*>(pf_router_kernel), dim3((N + kPfRouterTok - 1) / kPfRouterTok, (E + 15) / 16),
               dim3(256), r_smem, s, &ra);
    MOEB_CUDA(cudaGetLastError());
    PfTopkArgs ta{};
    ta.logits = S->pf_logits.p;
    ta.scores = S->pf_scores.p;
    ta.sel = S->pf_sel.p;
    ta.wts = S->pf_wts.p;
    ta.slot_w = Sh ? S->pf_slot_w.p : nullptr;
    ta.cnt = S->pf_cnt.p;
    ta.N = N;
    ta.E = E;
    ta.k = k;
    ta.renormalize = S->model.renormalize;
    ta.shared_gate = S->model.shared_gate;
    ta.routed_scale = S->model.routed_scale;
    ta.plan.cnt = S->pf_cnt.p;
    ta.plan.cursor = S->pf_cursor.p;
    ta.plan.ls = S->layers.p + l;
    ta.plan.slot_base = reinterpret_cast<const unsigned char*>(S->slots.p + (size_t)l * S->slots_alloc * S->expert_elems);
    ta.plan.stage_base = S->pf_stage.p ? reinterpret_cast<const unsigned char*>(S->pf_stage.p) + (size_t)(l % 2) * E * eb
                                  : nullptr;
    ta.plan.shared_w = Sh ? reinterpret_cast<const unsigned char*>(S->shared_w.p + (size_t)l * 3 * Sh * d) : nullptr;
    ta.plan.tiled_base = retile ? reinterpret_cast<const unsigned char*>(S->pf_tiled.p) : nullptr;
    if (retile && Sh) ta.plan.shared_w = reinterpret_cast<const unsigned char*>(S->pf_tiled.p + (size_t)E * S->expert_elems);
    ta.plan.expert_bytes = eb;
    ta.plan.N = N;
    ta.plan.E = E;
    ta.plan.d = d;
    ta.plan.F = F;
    ta.plan.S = Sh;
    ta.plan.items = S->pf_items.p;
    ta.plan.hdr = S->pf_hdr.p;
    ta.ticket = S->pf_cnt.p + kMaxE;
    launch_pdl(reinterpret_cast<const void*>(pf_topk_kernel), dim3((N + 7) / 8), dim3(256), 0, s, &ta);
    MOEB_CUDA(cudaGetLastError());
    PfScatterArgs sa{};
    sa.sel = S->pf_sel.p;
    sa.wts = S->pf_wts.p;
    sa.u = S->pf_u.p;
    sa.cursor = S->pf_cursor.p;
    sa.slot_w = S->pf_slot_w.p;
    sa.entry_slot = S->pf_entry.p;
    sa.xg = S->pf_xg.p;
    sa.N = N;
    sa.k = k;
    sa.d = d;
    sa.R = S->pf_R;
    sa.ctr_zero = S->pf_ctr.p;
    sa.n_ctr = (uint32_t)S->pf_ctr.n;
    launch_pdl(reinterpret_cast<const void*>(pf_scatter_kernel), dim3((N * k + 31) / 32), dim3(256), 0, s, &sa);
    MOEB_CUDA(cudaGetLastError());
    if (retile) {
      PfRetileArgs rt{};
      rt.ls = S->layers.p + l;
      rt.slot_base = ta.plan.slot_base;
      rt.stage_base = ta.plan.stage_base;
      rt.shared_src = Sh ? reinterpret_cast<const unsigned char*>(S->shared_w.p + (size_t)l * 3 * Sh * d) : nullptr;
      rt.dst = reinterpret_cast<unsigned char*>(S->pf_tiled.p);
      rt.expert_bytes = eb;
      rt.E = E;
      rt.d = d;
      rt.F = F;
      rt.S = Sh;
      const uint32_t Fm = std::max(F, Sh), tiles = (Fm / 128) * (d / 64) * 2 + (d / 128) * (Fm / 64);
      launch_pdl(reinterpret_cast<const void*>(pf_retile_kernel), dim3(tiles, E + (Sh ? 1 : 0)), dim3(256), 0, s, &rt);
      MOEB_CUDA(cudaGetLastError());
    }
    PfGemmArgs ga{};
    ga.items = S->pf_items.p;
    ga.hdr = S->pf_hdr.p;
    ga.xg = S->pf_xg.p;
    ga.hg = S->pf_hg.p;
    ga.out = S->pf_out.p;
    ga.slot_w = S->pf_slot_w.p;
    ga.ctr = S->pf_ctr.p;
    ga.d = d;
    ga.R = S->pf_R;
    launch_pdl(reinterpret_cast<const void*>(pf_gemm_kernel), dim3(n_sm), dim3(kPfThreads), kPfStages * kPfStageBytes + 1024, s,
               &ga);
    MOEB_CUDA(cudaGetLastError());
    if (any_up) MOEB_CUDA(cudaEventRecord(S->pf_free[l % 2], s));
    float* ylog = log && N <= S->pf_log_n ? S->pf_log_y.p + (size_t)l * N * d : nullptr;
    {
      cudaLaunchConfig_t cc{};
      cc.gridDim = dim3((unsigned)std::min<uint64_t>(((uint64_t)N * d / 4 + 255) / 256, (uint64_t)n_sm * 16));
      cc.blockDim = dim3(256);
      cc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = kUsePdl ? 1 : 0;
      cc.attrs = at;
      cc.numAttrs = 1;
      const float* pout = S->pf_out.p;
      const int32_t* pent = S->pf_entry.p;
      MOEB_CUDA(cudaLaunchKernelEx(&cc, pf_combine_kernel, xin, pout, pent, xout, ylog, N, d, k, Sh ? 1u : 0u));
    }
    MOEB_CUDA(cudaGetLastError());
    if (ylog) {
      MOEB_CUDA(cudaMemcpyAsync(S->pf_log_x.p + (size_t)l * N * d, xin, (size_t)N * d * 2, cudaMemcpyDeviceToDevice, s));
      MOEB_CUDA(cudaMemcpyAsync(S->pf_log_scores.p + (size_t)l * N * E, S->pf_scores.p, (size_t)N * E * 4,
                                cudaMemcpyDeviceToDevice, s));
      MOEB_CUDA(cudaMemcpyAsync(S->pf_log_sel.p + (size_t)l * N * k, S->pf_sel.p, (size_t)N * k, cudaMemcpyDeviceToDevice, s));
    }
  }
  if (log) S->pf_last_n = N;
  return h2d;
}

// The device raises g_spin_timeout when a bounded wait gives up. It is read
// and cleared together: the failure is reported once (by the moeb_sync that
// observes it) and does not poison later syncs of this or other stacks.
static uint32_t take_spin_timeout() {
  uint32_t v = 0;
  cudaMemcpyFromSymbol(&v, g_spin_timeout, sizeof v);
  if (v) {
    const uint32_t zero = 0;
    cudaMemcpyToSymbol(g_spin_timeout, &zero, sizeof zero);
  }
  return v;
}

// The per-step logs hold the first rec_cap layer-steps since create; a
// longer run fails loudly instead of returning a silently truncated log.
static void check_log_capacity(const moeb_stack* s, uint64_t seq) {
  if (seq > s->rec_cap)
    throw Error(4, "decision log overflow: " + std::to_string(seq) + " layer-steps since create exceed the log "
                   "capacity of " + std::to_string(s->rec_cap));
}

}  // namespace moeb

extern "C" {

int moeb_create(const moeb_config* cfg, const moeb_model* model, const void* weights_host, int device,
                moeb_stack** out) {
  return guarded([&] {
    auto* S = new moeb_stack();
    try {
      build_stack(S, *cfg, *model, weights_host, device);
    } catch (...) {
      delete S;
      throw;
    }
    *out = S;
  });
}

void moeb_destroy(moeb_stack* s) { delete s; }

int moeb_set_logits_trace(moeb_stack* s, const float* logits, uint64_t n_steps, uint64_t total_iterations) {
  return guarded([&] {
    MOEB_CUDA(cudaSetDevice(s->device));
    MOEB_CUDA(cudaStreamSynchronize(s->stream));
    if (logits && n_steps && s->predictor)
      throw Error(1, "the predictor needs weight-driven routing (no logits trace)");
    if (!logits || n_steps == 0) {
      s->trace.free();
      s->trace_steps = 0;
      s->total_iters = ~0ull;
      return;
    }
    const size_t n = (size_t)n_steps * s->L * s->B * s->E;
    s->trace.alloc(n);
    MOEB_CUDA(cudaMemcpy(s->trace.p, logits, n * sizeof(float), cudaMemcpyDefault));
    s->trace_steps = n_steps;
    s->total_iters = total_iterations ? total_iterations : ~0ull;
  });
}

int moeb_step(moeb_stack* s, const void* x, void* y, uint32_t B, void* stream) {
  return guarded([&] { step_stack(s, x, y, B, static_cast<cudaStream_t>(stream)); });
}

int moeb_prefill(moeb_stack* s, const void* x, void* y, uint32_t n_tokens, void* stream, uint64_t* h2d_bytes) {
  return guarded([&] {
    if (s->copier_error) throw Error(5, s->copier_msg);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
    MOEB_CUDA(cudaSetDevice(s->device));
    DeviceOrder& o = device_order(s->device);
    std::lock_guard<std::mutex> lk(o.mu);
    if (!o.ev) MOEB_CUDA(cudaEventCreateWithFlags(&o.ev, cudaEventDisableTiming));
    if (o.owner && o.owner != s) MOEB_CUDA(cudaStreamWaitEvent(st, o.ev, 0));
    const uint64_t b = prefill_stack(s, x, y, n_tokens, st);
    MOEB_CUDA(cudaEventRecord(o.ev, st));
    o.owner = s;
    if (h2d_bytes) *h2d_bytes = b;
  });
}

int moeb_get_prefill_log(moeb_stack* s, uint32_t layer, uint32_t* n_tokens, uint16_t* x_in, float* scores,
                         uint8_t* sel, float* y) {
  return guarded([&] {
    if (!s->rec_cap) throw Error(1, "prefill log needs MOEB_MODEL_LOG_STEPS");
    if (!s->pf_last_n) throw Error(1, "no prefill has run");
    if (layer >= s->L) throw Error(1, "layer out of range");
    MOEB_CUDA(cudaSetDevice(s->device));
    MOEB_CUDA(cudaDeviceSynchronize());
    const size_t N = s->pf_last_n, d = s->d, E = s->E, k = s->cfg.top_k;
    if (n_tokens) *n_tokens = (uint32_t)N;
    if (x_in) MOEB_CUDA(cudaMemcpy(x_in, s->pf_log_x.p + layer * N * d, N * d * 2, cudaMemcpyDeviceToHost));
    if (scores) MOEB_CUDA(cudaMemcpy(scores, s->pf_log_scores.p + layer * N * E, N * E * 4, cudaMemcpyDeviceToHost));
    if (sel) MOEB_CUDA(cudaMemcpy(sel, s->pf_log_sel.p + layer * N * k, N * k, cudaMemcpyDeviceToHost));
    if (y) MOEB_CUDA(cudaMemcpy(y, s->pf_log_y.p + layer * N * d, N * d * 4, cudaMemcpyDeviceToHost));
  });
}

int moeb_sync(moeb_stack* s) {
  return guarded([&] {
    MOEB_CUDA(cudaSetDevice(s->device));
    MOEB_CUDA(cudaStreamSynchronize(s->stream));
    MOEB_CUDA(cudaDeviceSynchronize());
    // and every upload the steps published (prefetches for later steps
    // included) has been issued by the copy thread and has landed
    if (s->host_seq) drain_uploads(s);
    const uint32_t to = take_spin_timeout();
    if (s->copier_error) throw Error(5, s->copier_msg);  // a failed upload is the cause of any stall
    if (to) throw Error(5, "device wait timed out (code " + std::to_string(to) + "): upload pipeline stalled");
  });
}

int moeb_get_metrics(moeb_stack* s, moeb_metrics* m) {
  return guarded([&] {
    MOEB_CUDA(cudaDeviceSynchronize());
    EngineState st;
    MOEB_CUDA(cudaMemcpy(&st, s->st.p, sizeof st, cudaMemcpyDeviceToHost));
    metrics_from_counters(*m, st.c, st.it, st.now);
  });
}

int moeb_get_decisions_json(moeb_stack* s, char** json) {
  return guarded([&] {
    if (!s->rec_cap) throw Error(4, "stack was created without MOEB_MODEL_LOG_STEPS");
    MOEB_CUDA(cudaDeviceSynchronize());
    EngineState st;
    MOEB_CUDA(cudaMemcpy(&st, s->st.p, sizeof st, cudaMemcpyDeviceToHost));
    check_log_capacity(s, st.seq);
    const size_t n = std::min<uint64_t>(st.seq, s->rec_cap);
    std::vector<StepRec> r(n);
    std::vector<TokRec> t(n * s->B);
    if (n) {
      MOEB_CUDA(cudaMemcpy(r.data(), s->recs.p, n * sizeof(StepRec), cudaMemcpyDeviceToHost));
      MOEB_CUDA(cudaMemcpy(t.data(), s->toks.p, n * s->B * sizeof(TokRec), cudaMemcpyDeviceToHost));
    }
    const std::string js = steps_json(r.data(), t.data(), n, s->B);
    char* p = static_cast<char*>(std::malloc(js.size() + 1));
    std::memcpy(p, js.c_str(), js.size() + 1);
    *json = p;
  });
}

static_assert(sizeof(moeb_step_record) == sizeof(StepRec) && offsetof(moeb_step_record, load) == offsetof(StepRec, load) &&
                  offsetof(moeb_step_record, evict_expert) == offsetof(StepRec, ev_e),
              "moeb_step_record mirrors the device StepRec");
static_assert(sizeof(moeb_token_record) == sizeof(TokRec) && offsetof(moeb_token_record, kept) == offsetof(TokRec, kept),
              "moeb_token_record mirrors the device TokRec");

int moeb_get_decisions(moeb_stack* s, moeb_step_record* steps, moeb_token_record* toks, size_t cap_steps,
                       size_t* n_steps) {
  return guarded([&] {
    if (!s->rec_cap) throw Error(4, "stack was created without MOEB_MODEL_LOG_STEPS");
    MOEB_CUDA(cudaDeviceSynchronize());
    EngineState st;
    MOEB_CUDA(cudaMemcpy(&st, s->st.p, sizeof st, cudaMemcpyDeviceToHost));
    check_log_capacity(s, st.seq);
    const size_t n = st.seq;
    *n_steps = n;
    const size_t k = std::min(n, cap_steps);
    if (steps && k) MOEB_CUDA(cudaMemcpy(steps, s->recs.p, k * sizeof(StepRec), cudaMemcpyDeviceToHost));
    if (toks && k) MOEB_CUDA(cudaMemcpy(toks, s->toks.p, k * s->B * sizeof(TokRec), cudaMemcpyDeviceToHost));
  });
}

int moeb_get_scores(moeb_stack* s, float* out, size_t cap, size_t* n) {
  return guarded([&] {
    if (!s->rec_cap) throw Error(4, "stack was created without MOEB_MODEL_LOG_STEPS");
    MOEB_CUDA(cudaDeviceSynchronize());
    EngineState st;
    MOEB_CUDA(cudaMemcpy(&st, s->st.p, sizeof st, cudaMemcpyDeviceToHost));
    check_log_capacity(s, st.seq);
    const size_t total = std::min<uint64_t>(st.seq, s->rec_cap) * s->B * s->E;
    const size_t k = std::min(total, cap);
    if (k) MOEB_CUDA(cudaMemcpy(out, s->scores_log.p, k * sizeof(float), cudaMemcpyDeviceToHost));
    *n = total;
  });
}

int moeb_get_copy_times(moeb_stack* s, float* ms, size_t cap, size_t* n) {
  return guarded([&] {
    MOEB_CUDA(cudaStreamSynchronize(s->copy_stream));
    std::lock_guard<std::mutex> g(s->io_mu);
    for (int i = 0; i < moeb_stack::kEv; ++i) s->harvest(i);
    *n = s->io.per_copy_ms.size();
    if (ms) std::memcpy(ms, s->io.per_copy_ms.data(), std::min(cap, *n) * sizeof(float));
  });
}

int moeb_get_pred_scores(moeb_stack* s, float* out, size_t cap, size_t* n) {
  return guarded([&] {
    if (!s->predictor || !s->rec_cap)
      throw Error(4, "stack was created without MOEB_MODEL_PREDICTOR | MOEB_MODEL_LOG_STEPS");
    MOEB_CUDA(cudaDeviceSynchronize());
    EngineState st;
    MOEB_CUDA(cudaMemcpy(&st, s->st.p, sizeof st, cudaMemcpyDeviceToHost));
    check_log_capacity(s, st.seq);
    const size_t total = std::min<uint64_t>(st.seq, s->rec_cap) * s->B * s->E;
    const size_t k = std::min(total, cap);
    if (out && k) MOEB_CUDA(cudaMemcpy(out, s->pred_log.p, k * sizeof(float), cudaMemcpyDeviceToHost));
    *n = total;
  });
}

int moeb_get_io_stats(moeb_stack* s, moeb_io_stats* out) {
  return guarded([&] {
    MOEB_CUDA(cudaStreamSynchronize(s->copy_stream));
    std::lock_guard<std::mutex> g(s->io_mu);
    for (int i = 0; i < moeb_stack::kEv; ++i) s->harvest(i);
    out->h2d_bytes = s->io.h2d_bytes;
    out->h2d_copies = s->io.h2d_copies;
    out->d2d_copies = s->io.d2d_copies;
    out->steps = s->io.steps;
    out->copy_ms = s->io.copy_ms + (s->io.timed_uploads ? s->io.upload_ms * (double)s->io.h2d_copies /
                                                             (double)s->io.timed_uploads : 0.0);
    out->spec_jobs = s->io.spec_jobs;
    out->spec_promoted = s->io.spec_promoted;
    out->spec_chunks = s->io.spec_chunks;
    out->spec_bytes = s->io.spec_bytes;
  });
}

int moeb_get_layer_outputs(moeb_stack* s, float* out, size_t cap) {
  return guarded([&] {
    MOEB_CUDA(cudaDeviceSynchronize());
    const size_t n = std::min<size_t>(cap, (size_t)s->L * s->B * s->d);
    MOEB_CUDA(cudaMemcpy(out, s->y_layers.p, n * sizeof(float), cudaMemcpyDeviceToHost));
  });
}

int moeb_reset(moeb_stack* s) {
  return guarded([&] {
    MOEB_CUDA(cudaSetDevice(s->device));
    MOEB_CUDA(cudaStreamSynchronize(s->stream));
    MOEB_CUDA(cudaStreamSynchronize(s->copy_stream));
    reset_state(s, s->stream);
    s->host_it = 0;
    take_spin_timeout();
  });
}

int moeb_get_kernel_stats(moeb_stack* s, moeb_kernel_stats* out) {
  return guarded([&] {
    MOEB_CUDA(cudaSetDevice(s->device));
    MOEB_CUDA(cudaStreamSynchronize(s->stream));
    if (s->timing) s->tk_harvest_all();
    EngineState st;
    MOEB_CUDA(cudaMemcpy(&st, s->st.p, sizeof st, cudaMemcpyDeviceToHost));
    *out = moeb_kernel_stats{};
    out->route_ms = s->kern_ms[0];
    out->ffn_ms = s->kern_ms[1];
    out->route_launches = s->n_launch_layers;
    out->ffn_launches = s->n_launch_layers;
    out->ffn_bytes = st.ffn_bytes;
    out->ffn_planned = st.ffn_launches;
    for (int i = 0; i < 32; ++i) out->prof_ns[i] = st.prof[i];
    const uint64_t gb = (uint64_t)s->E * s->d * 2 + 2ull * s->B * s->d * 2 + (uint64_t)s->B * (s->E + 1) * 4 +
                        (s->model.shared_gate ? (uint64_t)s->d * 2 : 0);
    out->route_bytes = gb * s->n_launch_layers;
  });
}

int moeb_reset_kernel_stats(moeb_stack* s) {
  return guarded([&] {
    MOEB_CUDA(cudaStreamSynchronize(s->stream));
    if (s->timing) s->tk_harvest_all();
    for (int k = 0; k < 2; ++k) { s->kern_ms[k] = 0; s->kern_n[k] = 0; }
    s->n_launch_layers = 0;
    EngineState st;
    MOEB_CUDA(cudaMemcpy(&st, s->st.p, sizeof st, cudaMemcpyDeviceToHost));
    st.ffn_bytes = 0;
    st.ffn_launches = 0;
    MOEB_CUDA(cudaMemcpy(s->st.p, &st, sizeof st, cudaMemcpyHostToDevice));
    std::lock_guard<std::mutex> g(s->io_mu);
    MOEB_CUDA(cudaStreamSynchronize(s->copy_stream));
    for (int i = 0; i < moeb_stack::kEv; ++i) s->harvest(i);
    s->io = IoAcc{};
  });
}

void* moeb_stream(moeb_stack* s) { return s->stream; }

int moeb_get_timeline(moeb_stack* s, uint64_t* out, size_t cap, size_t* n) {
  return guarded([&] {
    if (!s->timeline.p) throw Error(1, "timeline: create the stack with MOEB_MODEL_TRACE_TIMELINE");
    MOEB_CUDA(cudaStreamSynchronize(s->stream));
    const size_t have = (size_t)std::min<uint64_t>(s->host_seq, 16384) * kTlWords;
    *n = have;
    if (out) MOEB_CUDA(cudaMemcpy(out, s->timeline.p, std::min(cap, have) * 8, cudaMemcpyDeviceToHost));
  });
}

int moeb_set_expert_sources(moeb_stack* s, const void* const* ptrs, size_t n) {
  return guarded([&] {
    MOEB_CUDA(cudaSetDevice(s->device));
    MOEB_CUDA(cudaDeviceSynchronize());
    drain_uploads(s);  // no upload issued or in flight while the table changes
    if (!ptrs) {
      std::lock_guard<std::mutex> g(s->io_mu);
      s->src_tab.clear();
      s->serial = s->serial_at_create;
      return;
    }
    if (n != (size_t)s->L * s->E) throw Error(1, "expert sources: need one pointer per (layer, expert)");
    std::vector<const char*> tab(n);
    for (size_t i = 0; i < n; ++i) {
      cudaPointerAttributes at{};
      MOEB_CUDA(cudaPointerGetAttributes(&at, ptrs[i]));
      if (at.type != cudaMemoryTypeDevice) throw Error(1, "expert sources: every pointer must be device memory");
      if (at.device != s->device) {
        int ok = 0;
        MOEB_CUDA(cudaDeviceCanAccessPeer(&ok, s->device, at.device));
        if (!ok) throw Error(1, "expert sources: no peer access to device " + std::to_string(at.device));
        const cudaError_t pe = cudaDeviceEnablePeerAccess(at.device, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) MOEB_CUDA(pe);
        cudaGetLastError();
      }
      tab[i] = static_cast<const char*>(ptrs[i]);
    }
    std::lock_guard<std::mutex> g(s->io_mu);
    s->src_tab = std::move(tab);
    // Measured: with the pipelined schedule (the FFN spinning on copies_done)
    // a device-to-device upload issued by the copy thread does not complete
    // while the FFN waits for it, although a standalone device-to-device copy
    // does run beside a kernel that fills every SM (tools/probe/d2d_ce_probe.cu).
    // So with a device tier the stack orders uploads on the host (serial mode:
    // the compute stream waits for each step's copies before its FFN).
    // MOEB_TIER_PIPELINED=1 keeps the pipelined schedule (diagnostics).
    if (!getenv("MOEB_TIER_PIPELINED")) s->serial = true;
  });
}

int moeb_debug_ffn_tstamps(moeb_stack* s, uint64_t* out, size_t cap, size_t* n) {
  return guarded([&] {
    MOEB_CUDA(cudaDeviceSynchronize());
    *n = s->ffn_ts.n;
    if (out && *n) MOEB_CUDA(cudaMemcpy(out, s->ffn_ts.p, std::min(cap, *n) * 8, cudaMemcpyDeviceToHost));
  });
}

int moeb_get_host_pool(moeb_stack* s, const void** pool, size_t* expert_bytes) {
  *pool = s->pool;
  *expert_bytes = s->expert_elems * 2;
  return 0;
}

int moeb_host_pool_flags(moeb_stack* s, uint32_t* flags) {
  *flags = s->layout_flags();
  return 0;
}

}  // extern "C"
