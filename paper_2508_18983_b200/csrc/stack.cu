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
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/moesched_b200.h"
#include "decide.cuh"
#include "engine_host.h"
#include "host_common.h"
#include "layer.cuh"
#include "weights.cuh"

namespace moeb {

constexpr int kMaxCmds = 3 * kMaxE + 8;
constexpr uint32_t kRing = 256;

struct MailCmd {
  uint64_t src_off;   // byte offset into the pinned host pool
  uint64_t dst;       // device address
  uint64_t bytes;
  uint32_t id;        // upload id; copies_done := id after the copy
  uint32_t wait_ffn;  // nonzero: copy waits for ffn_done >= wait_ffn
};
struct MailEntry {
  volatile uint64_t seq;
  uint32_t n, pad;
  MailCmd cmd[kMaxCmds];
};

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
  uint32_t* ffn_ctr;
  MailEntry* ring;
  const volatile uint64_t* host_ack;
  float* scores_log;          // [rec_cap][B][E] or null
  StepRec* recs;
  TokRec* toks;
  uint64_t rec_cap;
};

struct DecideKSmem {
  DecideSmem d;
  NextSmem n;
  StepScratch s;
  DevCfg cfg;
  float sc[kMaxB][kMaxE];
  float nsc[kMaxB][kMaxE];
  float sg[kMaxB];
  float denom[kMaxB];
  uint64_t it, seq;
};

__device__ __forceinline__ uint16_t* slot_ptr(const DecideArgs& a, uint32_t layer, int slot) {
  return a.slots + ((size_t)layer * a.slots_alloc + (uint32_t)slot) * a.expert_elems;
}

__global__ void __launch_bounds__(kThreads, 1) decide_kernel(DecideArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DecideKSmem* sm = reinterpret_cast<DecideKSmem*>(smem_raw);
  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    sm->cfg = a.cfg;
    sm->it = a.st->it;
    sm->seq = a.st->seq + 1;
  }
  __syncthreads();
  const DevCfg& cfg = sm->cfg;
  const uint32_t B = cfg.B, E = cfg.E, L = cfg.L, layer = a.layer;
  const uint64_t it = sm->it;
  uint64_t tit = it;
  uint32_t tl = layer + 1;
  if (tl == L) { tl = 0; ++tit; }
  const bool has_target = tit < a.total_iters;
  const bool want_next = cfg.pre && has_target && a.trace;
  for (uint32_t t = warp; t < B; t += kWarps) {
    const float* lg = a.trace ? a.trace + (((it % a.trace_steps) * L + layer) * B + t) * E
                              : a.logits + (size_t)t * (E + 1);
    softmax_warp(lg, E, sm->sc[t]);
    if (want_next) {
      const float* nl = a.trace + (((tit % a.trace_steps) * L + tl) * B + t) * E;
      softmax_warp(nl, E, sm->nsc[t]);
    }
    if (lane == 0 && a.shared_gate) {
      const float z = a.logits[(size_t)t * (E + 1) + E];
      sm->sg[t] = __fdiv_rn(1.0f, 1.0f + expf(-z));
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < B * E; i += blockDim.x) {
    const uint32_t t = i / E, e = i % E;
    sm->d.s[t][e] = (double)sm->sc[t][e];
    if (want_next) { sm->d.ns[t][e] = (double)sm->nsc[t][e]; sm->d.np[t][e] = 0.0; }
    if (a.scores_log && sm->seq <= a.rec_cap) a.scores_log[((sm->seq - 1) * B + t) * E + e] = sm->sc[t][e];
  }
  if (threadIdx.x == 0) sm->d.next_has_pred = 0;
  __syncthreads();

  StepCtx cx;
  cx.cfg = &cfg;
  cx.st = a.st;
  cx.layers = a.layers;
  cx.hist = a.hist;
  cx.logs = nullptr;
  cx.it = it;
  cx.layer = layer;
  cx.has_target = want_next ? 1u : 0u;
  cx.target_layer = tl;
  cx.target_it = tit;
  StepRec* rec = nullptr;
  TokRec* toks = nullptr;
  if (a.recs && sm->seq <= a.rec_cap) {
    rec = a.recs + (sm->seq - 1);
    toks = a.toks + (sm->seq - 1) * B;
  }
  decide_step(cx, &sm->d, &sm->n, &sm->s, rec, toks);
  __syncthreads();

  // ---------------------------------------------------------------- plan
  DecideSmem* d = &sm->d;
  const StepOut& out = d->out;
  if (threadIdx.x < 32 * 2 && threadIdx.x < B) {
    // combine-weight denominators (Mixtral renormalisation)
    const uint32_t t = threadIdx.x;
    float s = 0.f;
    for (uint32_t i = 0; i < d->nsel[t]; ++i) s += sm->sc[t][d->sel[t][i]];
    sm->denom[t] = s;
  }
  for (uint32_t i = threadIdx.x; i < kMaxItems + 2; i += blockDim.x) a.ffn_ctr[i] = 0;
  __syncthreads();
  if (threadIdx.x != 0) return;

  Plan* p = a.plan;
  MailEntry* me = &a.ring[sm->seq % kRing];
  // the ring slot must have been consumed by the copy thread
  {
    const uint64_t t0 = globaltimer_ns();
    while (sm->seq > kRing && *a.host_ack < sm->seq - kRing) {
      __nanosleep(1000);
      if (globaltimer_ns() - t0 > kSpinLimitNs) { atomicExch(&g_spin_timeout, 4u); break; }
    }
  }
  uint32_t n_items = 0, n_cmds = 0;
  EngineState* st = a.st;
  LayerState* ls = &a.layers[layer];
  auto add_item = [&](const uint16_t* w, uint32_t F, uint32_t wait, uint32_t kind, uint32_t e) {
    Item& itm = p->items[n_items++];
    itm.w = w;
    itm.F = F;
    itm.wait = wait;
    itm.kind = kind;
    itm.expert = e;
    uint32_t n = 0;
    for (uint32_t t = 0; t < B; ++t) {
      bool sel = false;
      if (kind == 0) {
        sel = true;
      } else {
        for (uint32_t i = 0; i < d->nsel[t]; ++i) sel |= d->sel[t][i] == e;
      }
      if (!sel) continue;
      float wt;
      if (kind == 0) {
        wt = a.shared_gate ? sm->sg[t] : 1.0f;
      } else {
        wt = sm->sc[t][e];
        if (a.renormalize) wt = __fdiv_rn(wt, sm->denom[t]);
        wt = __fmul_rn(wt, a.routed_scale);
      }
      itm.tok[n] = (uint8_t)t;
      itm.wt[n] = wt;
      ++n;
    }
    itm.n_tok = n;
  };
  auto add_cmd = [&](uint32_t src_layer, uint32_t e, uint16_t* dst, uint32_t wait_ffn) -> uint32_t {
    const uint32_t id = ++st->next_copy;
    MailCmd& c = me->cmd[n_cmds++];
    c.src_off = ((uint64_t)src_layer * E + e) * a.expert_elems * 2;
    c.dst = (uint64_t)dst;
    c.bytes = a.expert_elems * 2;
    c.id = id;
    c.wait_ffn = wait_ffn;
    return id;
  };
  if (a.shared_w) add_item(a.shared_w, a.S, 0, 0, 0);
  // residents: ready ones first, then those whose (prefetch) upload is in flight
  for (int pass = 0; pass < 2; ++pass) {
    for (uint32_t i = 0; i < out.n_res; ++i) {
      const uint32_t e = out.res[i];
      const int slot = out.res_slot[i];
      const uint32_t wait = ls->slot_copy[slot];
      if ((wait == 0) != (pass == 0)) continue;
      add_item(slot_ptr(a, layer, slot), a.F, wait, 1, e);
    }
  }
  // the resident items that wait keep upload order (ids ascending)
  uint32_t n_ready = 0;
  while (n_ready < n_items && p->items[n_ready].wait == 0) ++n_ready;
  for (uint32_t i = n_ready + 1; i < n_items; ++i) {
    Item x = p->items[i];
    uint32_t j = i;
    while (j > n_ready && p->items[j - 1].wait > x.wait) { p->items[j] = p->items[j - 1]; --j; }
    p->items[j] = x;
  }
  uint32_t si = 0;
  int8_t stage_of[kMaxE];
  for (uint32_t e = 0; e < E; ++e) stage_of[e] = -1;
  for (uint32_t i = 0; i < out.n_load; ++i) {
    const uint32_t e = out.load[i];
    const int slot = out.load_slot[i];
    uint16_t* dst;
    if (slot >= 0) {
      dst = slot_ptr(a, layer, slot);
    } else {
      stage_of[e] = (int8_t)si;
      dst = a.staging + (size_t)(si++ % a.n_stage) * a.expert_elems;
    }
    const uint32_t id = add_cmd(layer, e, dst, 0);
    if (slot >= 0) ls->slot_copy[slot] = id;
    add_item(dst, a.F, id, 2, e);
  }
  for (uint32_t i = 0; i < out.n_cpu; ++i) {
    const uint32_t e = out.cpu[i];
    uint16_t* dst = a.staging + (size_t)(si++ % a.n_stage) * a.expert_elems;
    const uint32_t id = add_cmd(layer, e, dst, 0);
    add_item(dst, a.F, id, 3, e);
  }
  uint32_t n_d2d = 0;
  for (uint32_t i = 0; i < out.n_def; ++i) {
    const uint32_t e = out.def_e[i];
    const int slot = out.def_slot[i];
    if (stage_of[e] < 0 || slot < 0) continue;
    p->d2d[n_d2d].src = a.staging + (size_t)stage_of[e] * a.expert_elems;
    p->d2d[n_d2d].dst = slot_ptr(a, layer, slot);
    ls->slot_copy[slot] = 0;  // filled by this step's FFN epilogue
    ++n_d2d;
  }
  for (uint32_t i = 0; i < out.n_pref; ++i) {
    const uint32_t e = out.pref[i];
    const int slot = out.pref_slot[i];
    const uint32_t tlayer = out.pref_layer;
    uint16_t* dst = slot >= 0 ? slot_ptr(a, tlayer, slot) : a.staging;
    const uint32_t id = add_cmd(tlayer, e, dst, (uint32_t)sm->seq);
    if (slot >= 0) a.layers[tlayer].slot_copy[slot] = id;
  }
  p->n_items = n_items;
  p->n_ready = n_ready;
  p->n_d2d = n_d2d;
  p->d2d_elems = a.expert_elems;
  p->seq = (uint32_t)sm->seq;
  me->n = n_cmds;
  __threadfence_system();
  me->seq = sm->seq;
  __threadfence_system();
  st->seq = sm->seq;
  if (layer == L - 1) st->it = it + 1;
}

// =================================================================== host

struct IoAcc {
  uint64_t h2d_bytes = 0, h2d_copies = 0, d2d_copies = 0, steps = 0;
  double copy_ms = 0.0;
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
  DevBuf<EngineState> st;
  DevBuf<LayerState> layers;
  DevBuf<double> hist;
  DevBuf<Plan> plan;
  DevBuf<uint32_t> ffn_ctr, copies_done, ffn_done;
  DevBuf<StepRec> recs;
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
  void (*ffn_fn)(FfnArgs) = nullptr;
  size_t ffn_smem = 0, gate_smem = 0, decide_smem = 0;
  std::mutex io_mu;
  IoAcc io;
  static constexpr int kEv = 512;
  cudaEvent_t ev_a[kEv] = {}, ev_b[kEv] = {};
  bool ev_live[kEv] = {};
  int ev_next = 0;

  void harvest(int i) {  // requires io_mu
    if (!ev_live[i]) return;
    cudaEventSynchronize(ev_b[i]);
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ev_a[i], ev_b[i]) == cudaSuccess) io.copy_ms += ms;
    ev_live[i] = false;
  }

  void copy_loop() {
    cudaSetDevice(device);
    CUdeviceptr done_ptr = (CUdeviceptr)copies_done.p;
    CUdeviceptr ffn_ptr = (CUdeviceptr)ffn_done.p;
    uint64_t expect = 1;
    unsigned spins = 0;
    while (!stop.load(std::memory_order_relaxed)) {
      MailEntry* me = &ring[expect % kRing];
      if (me->seq != expect) {
        if (++spins > 2000) std::this_thread::yield();
        continue;
      }
      spins = 0;
      std::atomic_thread_fence(std::memory_order_acquire);
      const uint32_t n = me->n;
      for (uint32_t i = 0; i < n; ++i) {
        const MailCmd c = me->cmd[i];
        if (c.wait_ffn &&
            cuStreamWaitValue32(copy_stream, ffn_ptr, c.wait_ffn, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
          copier_msg = "cuStreamWaitValue32 failed";
          copier_error = 5;
        }
        std::lock_guard<std::mutex> g(io_mu);
        const int ei = ev_next;
        ev_next = (ev_next + 1) % kEv;
        harvest(ei);
        cudaEventRecord(ev_a[ei], copy_stream);
        const cudaError_t ce = cudaMemcpyAsync(reinterpret_cast<void*>(c.dst),
                                               reinterpret_cast<const char*>(pool) + c.src_off, c.bytes,
                                               cudaMemcpyHostToDevice, copy_stream);
        cudaEventRecord(ev_b[ei], copy_stream);
        ev_live[ei] = true;
        if (ce != cudaSuccess) {
          copier_msg = std::string("upload failed: ") + cudaGetErrorString(ce);
          copier_error = 5;
        }
        if (cuStreamWriteValue32(copy_stream, done_ptr, c.id, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) {
          copier_msg = "cuStreamWriteValue32 failed";
          copier_error = 5;
        }
        io.h2d_bytes += c.bytes;
        io.h2d_copies += 1;
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
    for (int i = 0; i < kEv; ++i) {
      if (ev_a[i]) cudaEventDestroy(ev_a[i]);
      if (ev_b[i]) cudaEventDestroy(ev_b[i]);
    }
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

using FfnFn = void (*)(FfnArgs);
static FfnFn ffn_kernel_for(uint32_t B) {
  if (B <= 1) return ffn_kernel<1>;
  if (B <= 2) return ffn_kernel<2>;
  if (B <= 4) return ffn_kernel<4>;
  if (B <= 8) return ffn_kernel<8>;
  if (B <= 16) return ffn_kernel<16>;
  return ffn_kernel<32>;
}

static float fan_scale(uint32_t fan_in) { return (float)std::sqrt(3.0 / (double)fan_in); }

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
  int attr = 0;
  CUdevice cud;
  if (cuDeviceGet(&cud, device) == CUDA_SUCCESS &&
      cuDeviceGetAttribute(&attr, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR, cud) == CUDA_SUCCESS) {
    // stream memory operations are available on every sm_100 driver; the
    // attribute probe only initialises the driver API here
  }
  const cudaStream_t s = S->stream;
  const uint32_t L = S->L, E = S->E, B = S->B, d = S->d, F = S->F, Sh = S->S;
  const uint64_t seed = m.weight_seed;
  // resident (HBM) weights: router, shared expert, shared gate
  S->gate_w.alloc((size_t)L * E * d);
  for (uint32_t l = 0; l < L; ++l) synth(S->gate_w.p + (size_t)l * E * d, (uint64_t)E * d, seed, tid_router(l), 0, fan_scale(d), s);
  if (Sh) {
    S->shared_w.alloc((size_t)L * 3 * Sh * d);
    for (uint32_t l = 0; l < L; ++l) {
      uint16_t* base = S->shared_w.p + (size_t)l * 3 * Sh * d;
      synth(base, (uint64_t)Sh * d, seed, tid_shared(l, 0), 0, fan_scale(d), s);
      synth(base + (size_t)Sh * d, (uint64_t)Sh * d, seed, tid_shared(l, 1), 0, fan_scale(d), s);
      synth(base + 2 * (size_t)Sh * d, (uint64_t)Sh * d, seed, tid_shared(l, 2), 0, fan_scale(Sh), s);
    }
  }
  if (m.shared_gate) {
    S->sgate_w.alloc((size_t)L * d);
    for (uint32_t l = 0; l < L; ++l) synth(S->sgate_w.p + (size_t)l * d, d, seed, tid_shared_gate(l), 0, fan_scale(d), s);
  }
  // pinned host pool of every routed expert
  const uint64_t eb = S->expert_elems * 2;
  const uint64_t pool_bytes = (uint64_t)L * E * eb;
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
    // generate on the device, expert by expert, then D2H into the pool
    DevBuf<uint16_t> tmp(2 * S->expert_elems);
    for (uint64_t i = 0; i < (uint64_t)L * E; ++i) {
      const uint32_t l = (uint32_t)(i / E), e = (uint32_t)(i % E);
      uint16_t* buf = tmp.p + (i & 1) * S->expert_elems;
      synth(buf, (uint64_t)F * d, seed, tid_expert(l, e, 0), 0, fan_scale(d), s);
      synth(buf + (size_t)F * d, (uint64_t)F * d, seed, tid_expert(l, e, 1), 0, fan_scale(d), s);
      synth(buf + 2 * (size_t)F * d, (uint64_t)F * d, seed, tid_expert(l, e, 2), 0, fan_scale(F), s);
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
  // decision engine state
  std::vector<LayerState> ls;
  init_layers(S->dcfg, cfg.init_fill, cfg.seed, ls);
  EngineState st{};
  rng_seed(st.rng, derive_seed(cfg.seed, 0x94ed1c70ULL));
  S->st.alloc(1);
  S->layers.alloc(L);
  S->hist.alloc((size_t)L * cfg.window * E);
  S->hist.zero(s);
  MOEB_CUDA(cudaMemcpyAsync(S->st.p, &st, sizeof st, cudaMemcpyHostToDevice, s));
  MOEB_CUDA(cudaMemcpyAsync(S->layers.p, ls.data(), L * sizeof(LayerState), cudaMemcpyHostToDevice, s));
  // initial residency: upload the resident experts into their slots
  for (uint32_t l = 0; l < L; ++l)
    for (uint32_t e = 0; e < E; ++e)
      if (ls[l].slot_of[e] >= 0)
        MOEB_CUDA(cudaMemcpyAsync(S->slots.p + ((size_t)l * S->slots_alloc + ls[l].slot_of[e]) * S->expert_elems,
                                  reinterpret_cast<char*>(S->pool) + ((uint64_t)l * E + e) * eb, eb,
                                  cudaMemcpyHostToDevice, s));
  S->plan.alloc(1);
  S->ffn_ctr.alloc(kMaxItems + 2);
  S->ffn_ctr.zero(s);
  S->copies_done.alloc(1);
  S->copies_done.zero(s);
  S->ffn_done.alloc(1);
  S->ffn_done.zero(s);
  if (m.flags & MOEB_MODEL_LOG_STEPS) {
    S->rec_cap = 16384;
    S->recs.alloc(S->rec_cap);
    S->toks.alloc(S->rec_cap * B);
    S->scores_log.alloc(S->rec_cap * B * E);
  }
  MOEB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&S->ring), sizeof(MailEntry) * kRing, cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(S->ring, 0, sizeof(MailEntry) * kRing);
  MOEB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&S->ack), 64, cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(S->ack, 0, 64);
  // kernel resources
  S->gate_smem = (size_t)B * d * 2;
  S->ffn_smem = (size_t)B * d * 2;
  S->decide_smem = sizeof(DecideKSmem);
  MOEB_CUDA(cudaFuncSetAttribute(gate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->gate_smem));
  S->ffn_fn = ffn_kernel_for(B);
  MOEB_CUDA(cudaFuncSetAttribute(S->ffn_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->ffn_smem));
  MOEB_CUDA(cudaFuncSetAttribute(decide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->decide_smem));
  int sms = 0, occ = 0;
  MOEB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  MOEB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, S->ffn_fn, kFfnThreads, S->ffn_smem));
  if (occ < 1) throw Error(5, "ffn_kernel does not fit on an SM");
  S->ffn_grid = sms * occ;
  const uint32_t nW = (uint32_t)S->ffn_grid * kFfnWarps;
  if ((d + nW - 1) / nW > (uint32_t)kMaxRowsPerWarp) throw Error(1, "model: d_model too large for the FFN grid");
  MOEB_CUDA(cudaStreamSynchronize(s));
  S->copier = std::thread([S] { S->copy_loop(); });
}

static void step_stack(moeb_stack* S, const void* x, void* y, uint32_t B, cudaStream_t user) {
  if (B != S->B) throw Error(1, "step: batch must equal the configured batch_size");
  if (S->copier_error) throw Error(5, S->copier_msg);
  if (S->cfg.pre && !S->trace.p) throw Error(1, "stage Pre needs a logits trace (moeb_set_logits_trace)");
  cudaStream_t s = user ? user : S->stream;
  const uint32_t L = S->L, E = S->E, d = S->d;
  MOEB_CUDA(cudaMemcpyAsync(S->hidden.p, x, (size_t)B * d * 2, cudaMemcpyDeviceToDevice, s));
  int cur = 0;
  for (uint32_t l = 0; l < L; ++l) {
    GateArgs g{};
    g.x = S->hidden.p + (size_t)cur * B * d;
    g.wg = S->gate_w.p + (size_t)l * E * d;
    g.wsg = S->model.shared_gate ? S->sgate_w.p + (size_t)l * d : nullptr;
    g.u = S->u.p;
    g.logits = S->logits.p;
    g.B = B;
    g.d = d;
    g.E = E;
    const uint32_t rows = E + (g.wsg ? 1 : 0);
    gate_kernel<<<(rows + 1) / 2, kGateThreads, S->gate_smem, s>>>(g);
    MOEB_CUDA(cudaGetLastError());

    DecideArgs a{};
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
    a.ffn_ctr = S->ffn_ctr.p;
    uint64_t* ack_dev = nullptr;
    MailEntry* ring_dev = nullptr;
    MOEB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ring_dev), S->ring, 0));
    MOEB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ack_dev), S->ack, 0));
    a.ring = ring_dev;
    a.host_ack = ack_dev;
    a.scores_log = S->scores_log.p;
    a.recs = S->recs.p;
    a.toks = S->toks.p;
    a.rec_cap = S->rec_cap;
    decide_kernel<<<1, kThreads, S->decide_smem, s>>>(a);
    MOEB_CUDA(cudaGetLastError());

    FfnArgs f{};
    f.plan = S->plan.p;
    f.u = S->u.p;
    f.x_in = S->hidden.p + (size_t)cur * B * d;
    f.x_out = S->hidden.p + (size_t)(cur ^ 1) * B * d;
    f.y_out = S->y_layers.p + (size_t)l * B * d;
    f.h = S->h.p;
    f.ctr = S->ffn_ctr.p;
    f.copies_done = S->copies_done.p;
    f.ffn_done = S->ffn_done.p;
    f.B = B;
    f.d = d;
    f.Fmax = std::max(S->F, S->S);
    const uint32_t nW = (uint32_t)S->ffn_grid * kFfnWarps;
    f.rows_per_warp = (d + nW - 1) / nW;
    void* fargs[] = {&f};
    MOEB_CUDA(cudaLaunchKernel(S->ffn_fn, dim3(S->ffn_grid), dim3(kFfnThreads), fargs, S->ffn_smem, s));
    MOEB_CUDA(cudaGetLastError());
    cur ^= 1;
  }
  MOEB_CUDA(cudaMemcpyAsync(y, S->hidden.p + (size_t)cur * B * d, (size_t)B * d * 2, cudaMemcpyDeviceToDevice, s));
  std::lock_guard<std::mutex> g(S->io_mu);
  S->io.steps += 1;
}

static uint32_t read_spin_timeout() {
  uint32_t v = 0;
  cudaMemcpyFromSymbol(&v, g_spin_timeout, sizeof v);
  return v;
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

int moeb_sync(moeb_stack* s) {
  return guarded([&] {
    MOEB_CUDA(cudaSetDevice(s->device));
    MOEB_CUDA(cudaStreamSynchronize(s->stream));
    MOEB_CUDA(cudaDeviceSynchronize());
    if (const uint32_t to = read_spin_timeout()) {
      throw Error(5, "device wait timed out (code " + std::to_string(to) + "): upload pipeline stalled");
    }
    if (s->copier_error) throw Error(5, s->copier_msg);
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

int moeb_get_scores(moeb_stack* s, float* out, size_t cap, size_t* n) {
  return guarded([&] {
    if (!s->rec_cap) throw Error(4, "stack was created without MOEB_MODEL_LOG_STEPS");
    MOEB_CUDA(cudaDeviceSynchronize());
    EngineState st;
    MOEB_CUDA(cudaMemcpy(&st, s->st.p, sizeof st, cudaMemcpyDeviceToHost));
    const size_t total = std::min<uint64_t>(st.seq, s->rec_cap) * s->B * s->E;
    const size_t k = std::min(total, cap);
    if (k) MOEB_CUDA(cudaMemcpy(out, s->scores_log.p, k * sizeof(float), cudaMemcpyDeviceToHost));
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
    out->copy_ms = s->io.copy_ms;
  });
}

int moeb_get_layer_outputs(moeb_stack* s, float* out, size_t cap) {
  return guarded([&] {
    MOEB_CUDA(cudaDeviceSynchronize());
    const size_t n = std::min<size_t>(cap, (size_t)s->L * s->B * s->d);
    MOEB_CUDA(cudaMemcpy(out, s->y_layers.p, n * sizeof(float), cudaMemcpyDeviceToHost));
  });
}

int moeb_get_host_pool(moeb_stack* s, const void** pool, size_t* expert_bytes) {
  *pool = s->pool;
  *expert_bytes = s->expert_elems * 2;
  return 0;
}

}  // extern "C"
