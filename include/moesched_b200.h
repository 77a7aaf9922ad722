/*
 * moesched_b200.h — C-ABI of the B200-native MoE decode hot path.
 *
 * This is the drop-in boundary for the decision path of the reference
 * scheduler (/root/reference/proj/include/moesched/ headers). The reference is a
 * C++20 library with no FFI of its own; the entry points below are what a
 * foreign binding (ctypes / cgo / JNI) of that path binds, and what our C++
 * re-declaration of the reference headers (include/moesched/,
 * libmoesched.so) calls. Plain pointers and sizes only; no CUDA or torch
 * types cross this boundary (streams are opaque `void*` cudaStream_t).
 *
 * Status codes (every function returning int):
 *   0 ok, 1 config (ConfigError), 2 io (IoError), 3 cache (CacheError),
 *   4 logic (std::logic_error), 5 cuda. moeb_last_error() returns the message
 *   of the last failure on the calling thread (exact reference wording where
 *   the reference has one).
 *
 * Limits of the device engine: E <= 64 experts per layer (residency and
 * selection sets are 64-bit masks), top_k <= 16, batch <= 32 tokens per step,
 * slots_per_layer <= 64. Violations return 1 with a message.
 */
#ifndef MOESCHED_B200_H
#define MOESCHED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MOEB_OK = 0,
  MOEB_ECONFIG = 1,
  MOEB_EIO = 2,
  MOEB_ECACHE = 3,
  MOEB_ELOGIC = 4,
  MOEB_ECUDA = 5
};

/* SimConfig (core.hpp:94-106) flattened. policy: 0 ScoreWindow, 1 LRU.
 * init_fill: 0 FirstSlots, 1 SeededRandom, 2 Empty. queue_depth 0 = top_k. */
typedef struct moeb_config {
  uint32_t num_layers, experts, top_k, batch; /* ModelShape core.hpp:40-47 */
  double alpha;                               /* RouterConfig core.hpp:49-51 */
  uint32_t slots, window;                     /* CacheConfig core.hpp:56-61 */
  int32_t policy, init_fill;
  uint64_t t_attn, t_gpu, t_cpu_token, t_load, t_route; /* CostModel core.hpp:63-69 */
  double p_top, p_active;                     /* PredictorConfig core.hpp:71-75 */
  uint32_t queue_depth;
  int32_t ce, er, pre, ba;                    /* StageSet core.hpp:82-92 */
  uint64_t seed;
} moeb_config;

/* Real-layer dimensions (no reference counterpart: the reference abstracts
 * expert compute as t_gpu/t_load tasks, pipeline.cpp:229-259). */
typedef struct moeb_model {
  uint32_t d_model;      /* hidden size (multiple of 256) */
  uint32_t ffn;          /* routed expert intermediate size (multiple of 8) */
  uint32_t shared_ffn;   /* fused shared-expert intermediate size, 0 = none */
  int32_t shared_gate;   /* 1: Qwen2-MoE sigmoid gate on the shared expert */
  int32_t renormalize;   /* 1: Mixtral-style renormalised combine weights */
  float routed_scale;    /* DeepSeek routed_scaling_factor (1.0 for V2-Lite) */
  uint64_t weight_seed;  /* counter-based synthetic weights */
  uint32_t max_batch;    /* largest B a step will use (<= 32) */
  uint32_t flags;        /* MOEB_MODEL_* */
} moeb_model;

#define MOEB_MODEL_LOG_STEPS 1u     /* record per-step decision records */
#define MOEB_MODEL_TIME_KERNELS 2u  /* CUDA-event timing of every gate/decide/FFN launch */
#define MOEB_MODEL_TRACE_TIMELINE 4u /* device-clock timeline of every layer-step (moeb_get_timeline) */
/* Host pool layout: for batch > 1 each expert is [gate ffn x d][up ffn x d]
 * [down d x ffn] (the HF layouts); batch-1 stacks with d_model <= 2048 (the
 * split-K FFN) store it row-interleaved, [ffn][3][d]: gate row r, up row r,
 * down column r. A caller-supplied pool declares that layout with this flag. */
#define MOEB_MODEL_DOWN_T 8u
/* Host pool layout of batch 2..32 stacks whose ffn and shared_ffn are
 * multiples of 128 (the tensor-core FFN): every expert is a sequence of 16 KB
 * [128 x 64] bf16 tiles in the SWIZZLE_128B K-major order, gate_up
 * [ffn/128][d/64][gate | up] then down [d/128][ffn/128][2 K-blocks]. */
#define MOEB_MODEL_TILED 64u
/* Bitwise-reproducible layer outputs. Always the case now (the batch-1
 * split-K FFN deals its rows round-robin, a fixed assignment); the flag is
 * accepted for API stability. */
#define MOEB_MODEL_DETERMINISTIC 16u
/* weights_host is caller memory (e.g. a shared-memory segment every process
 * of a node maps) to be FILLED with the synthetic weights in this stack's
 * layout; later stacks then pass it without this flag (with
 * MOEB_MODEL_DOWN_T when moeb_host_pool_flags says so). */
#define MOEB_MODEL_FILL_POOL 32u
/* The paper's partial-forward predictor for stage Pre in
 * weight-driven mode (no logits trace): the FFN also emits the partial
 * forward x + shared expert + resident hits (no uploaded or BA-streamed
 * expert), the next layer's gate CTAs apply that layer's router to it, and
 * the next layer's decision step first runs the previous step's
 * schedule_prefetch with every token's prediction supplied
 * (prefetch.cpp:43-49) — the same state transition as the reference
 * (nothing happens between a step's prefetch and the next gate event).
 * PredictorStats count the heads against the true scores
 * (moeb_metrics.trace_supplied / head_top / head_active / head_inactive).
 * Batch-1 split-K and tensor-core FFN shapes only. */
#define MOEB_MODEL_PREDICTOR 128u

typedef struct moeb_engine moeb_engine; /* decision engine only (simulate path) */
typedef struct moeb_stack moeb_stack;   /* full MoE decode stack */

const char* moeb_last_error(void);
int moeb_device_count(int* n);

/* ---------------- library-level policy calls (router.hpp / cache.hpp /
 * balancer.hpp / prefetch.hpp re-exports, executed on the device) --------- */

/* classify (router.hpp:31 / router.cpp:41-71). Lists are in ranking order;
 * thr[4] = {beta, T, L, R}. */
int moeb_classify(const double* scores, uint32_t E, uint32_t k, double alpha, double* thr,
                  uint32_t* actives, uint32_t* top, uint32_t* n_top, uint32_t* low,
                  uint32_t* n_low, uint32_t* alt, uint32_t* n_alt);

/* route (router.hpp:67-70) and optionally coalesce_for_batching
 * (router.hpp:79-81) on one batch. Outputs per token t (k entries each):
 * sel[t*k..], subs as (dropped, chosen) pairs sub[t*2k..], kept[t*k..]. */
int moeb_route(const double* scores, uint32_t B, uint32_t E, const uint8_t* resident_mask,
               uint32_t k, double alpha, int32_t coalesce, uint32_t* sel, uint32_t* n_sel,
               uint32_t* sub, uint32_t* n_sub, uint32_t* kept, uint32_t* n_kept,
               uint32_t* top_set, uint32_t* n_top_set, uint32_t* pending, uint32_t* n_pending);

/* coalesce_for_batching over an existing RouteResult (in/out arrays as
 * moeb_route's outputs); thresholds: per token {beta, T, L, R} of the
 * RouteResult's Classification, used exactly as given. */
int moeb_coalesce(const double* scores, uint32_t B, uint32_t E, const uint8_t* resident_mask,
                  uint32_t k, const double* thresholds, uint32_t* sel, uint32_t* n_sel, uint32_t* sub,
                  uint32_t* n_sub, uint32_t* kept, uint32_t* n_kept, const uint32_t* top_set,
                  uint32_t n_top_set, uint32_t* pending, uint32_t* n_pending);

/* plain_top_k (router.hpp:84). */
int moeb_plain_top_k(const double* scores, uint32_t E, uint32_t k, uint32_t* out, uint32_t* n_out);

/* balance (balancer.hpp:39). */
int moeb_balance(const uint32_t* uid, const uint32_t* batch, uint32_t n, uint64_t t_cpu_token,
                 uint64_t t_load, uint32_t* load_list, uint32_t* n_load, uint32_t* cpu_list,
                 uint32_t* n_cpu, uint64_t* c_load, uint64_t* c_cpu);

/* predict_scores (prefetch.hpp:32-37). rng_state: xoshiro256** words,
 * advanced in place. supplied may be NULL. head_kind: 0 top, 1 active, 2 inactive. */
int moeb_predict_scores(const double* true_next, const double* supplied, uint32_t E,
                        double p_top, double p_active, uint32_t k, double alpha,
                        uint64_t* rng_state, double* out, uint32_t* head, int32_t* head_kind);

/* build_queue (prefetch.hpp:56-60). */
int moeb_build_queue(const double* predicted, const uint8_t* resident_mask, uint32_t E,
                     uint32_t depth, uint32_t* entries, uint32_t* n_entries);

/* ---------------- CacheState (cache.hpp:25-78) on the device ------------- */
typedef struct moeb_cache moeb_cache;
int moeb_cache_create(uint32_t layers, uint32_t E, uint32_t slots, uint32_t window,
                      int32_t policy, int32_t init_fill, uint64_t seed, moeb_cache** out);
void moeb_cache_destroy(moeb_cache* c);
int moeb_cache_resident(moeb_cache* c, uint32_t layer, uint32_t* out, uint32_t* n);
int moeb_cache_record(moeb_cache* c, uint32_t layer, const double* scores, uint32_t n);
int moeb_cache_window_average(moeb_cache* c, uint32_t layer, uint32_t e, double* out);
/* victim < 0: nothing evictable */
int moeb_cache_try_evict(moeb_cache* c, uint32_t layer, int64_t* victim);
int moeb_cache_shield(moeb_cache* c, uint32_t layer, uint32_t e);
int moeb_cache_unshield_layer(moeb_cache* c, uint32_t layer);
int moeb_cache_is_shielded(moeb_cache* c, uint32_t layer, uint32_t e, int32_t* out);
int moeb_cache_touch(moeb_cache* c, uint32_t layer, uint32_t e, uint64_t now);
/* returns 3 (CacheError) when every resident is shielded, 4 when already resident */
int moeb_cache_admit(moeb_cache* c, uint32_t layer, uint32_t e, uint64_t now, int64_t* evicted);

/* ---------------- simulate (pipeline.hpp:97) on the device ---------------
 * The whole run_layer decision state machine (pipeline.cpp:128-344) replayed
 * by one device kernel over a score trace. scores: [iters][L][B][E] fp64;
 * pred/has_pred optional ([iters][L][B][E] / [iters][L][B]). The result is
 * read back with moeb_result_* and released with moeb_result_free. */
typedef struct moeb_result moeb_result;
int moeb_simulate(const moeb_config* cfg, const double* scores, const double* pred,
                  const uint8_t* has_pred, uint64_t iters, int32_t record_steps,
                  moeb_result** out);
/* JSON view of a result (same schema as the oracle's; caller frees with moeb_free). */
int moeb_result_json(const moeb_result* r, char** json);
/* Raw views (valid until moeb_result_free). */
typedef struct moeb_metrics {
  double tpot, hit_rate, substitution_ratio;
  uint64_t demand_loads, prefetch_loads, cpu_computed, hits, misses, substitutions,
      low_score_kept, selections, iterations, total_time;
  uint64_t draws, trace_supplied, head_top, head_active, head_inactive, issued, cancelled;
} moeb_metrics;
int moeb_result_metrics(const moeb_result* r, moeb_metrics* m);
/* task: {resource, kind, expert_layer (-1 none), expert, start, end, layer, iteration} */
typedef struct moeb_task {
  uint8_t resource, kind;
  int16_t expert_layer;
  uint32_t expert;
  uint64_t start, end;
  uint32_t layer, pad;
  uint64_t iteration;
} moeb_task;
int moeb_result_tasks(const moeb_result* r, const moeb_task** tasks, size_t* n);
typedef struct moeb_window {
  uint64_t iteration;
  uint32_t layer, pad;
  uint64_t attn_end, route_end, completion;
  uint64_t selected; /* bitmask of distinct selected experts */
} moeb_window;
int moeb_result_windows(const moeb_result* r, const moeb_window** w, size_t* n);
typedef struct moeb_eviction {
  uint64_t time;
  uint32_t layer, expert;
} moeb_eviction;
int moeb_result_evictions(const moeb_result* r, const moeb_eviction** ev, size_t* n);
int moeb_result_iteration_completion(const moeb_result* r, const uint64_t** t, size_t* n);
int moeb_result_cache_final(const moeb_result* r, uint32_t layer, uint32_t* out, uint32_t* n);
void moeb_result_free(moeb_result* r);
void moeb_free(void* p);

/* ---------------- the MoE decode stack (new real-layer API) ---------------
 * weights_host: optional [L][E][3*ffn*d] bf16 routed-expert pool (gate_proj,
 * up_proj, down_proj of each expert, HF layouts). NULL = synthetic
 * counter-based weights generated from model->weight_seed. */
int moeb_create(const moeb_config* cfg, const moeb_model* model, const void* weights_host,
                int device, moeb_stack** out);
void moeb_destroy(moeb_stack* s);

/* Trace-driven router logits: [n_steps][L][B][E] fp32 (host or device
 * pointer; copied). Step i of the stack uses slice i % n_steps. The gate GEMV
 * still runs; routing uses these logits. NULL disables (weight-driven mode).
 * Stage Pre needs a logits trace (the predictor reads the next layer's true
 * scores, pipeline.cpp:414). total_iterations bounds prefetch at the trace
 * end exactly as simulate() does (pipeline.cpp:407). */
int moeb_set_logits_trace(moeb_stack* s, const float* logits, uint64_t n_steps,
                          uint64_t total_iterations);

/* One decode step (one token per sequence) through all L layers.
 * x, y: device pointers, bf16 [B][d]; stream: cudaStream_t or NULL (the
 * stack's own stream). Asynchronous; the copy thread issues expert uploads. */
int moeb_step(moeb_stack* s, const void* x, void* y, uint32_t B, void* stream);
/* Prefill (prompt pass): n_tokens tokens of one sequence through all L
 * layers (x, y: device pointers, bf16 [n_tokens][d]). Plain top-k routing
 * (plain_top_k, router.cpp:252-260: no substitution — the paper's prefill is
 * the traditional offloading path), every selected expert
 * computed as a grouped tcgen05 GEMM after a warp-aggregated token -> expert
 * permutation. Experts outside the capped cache are uploaded from the pinned
 * pool into a staging area, layer l+1's while layer l computes; the decode
 * state (cache, score windows, counters) is not changed. Needs the
 * UMMA-tiled layout (a stack with max_batch 2..32, ffn and shared_ffn
 * multiples of 128). Synchronises the stream once at entry (residency);
 * h2d_bytes (nullable) = bytes uploaded. */
int moeb_prefill(moeb_stack* s, const void* x, void* y, uint32_t n_tokens, void* stream,
                 uint64_t* h2d_bytes);
/* Expert tier: upload each (layer, expert) from a
 * device pointer — a peer GPU's HBM over NVLink (peer access is enabled
 * here; across processes, map the peer's allocation with CUDA IPC first), or
 * this GPU's — instead of the pinned host pool. ptrs: [L*E], each pointing to
 * that expert's weights in this stack's pool layout (moeb_host_pool_flags);
 * NULL restores the host pool. Call between steps (synchronises the device).
 * Decisions are unchanged; only where the upload bytes come from. A device
 * tier puts the stack's uploads in serial mode (the compute stream waits for
 * each step's uploads before its FFN): measured, a device-to-device upload
 * does not complete while the pipelined FFN spins waiting for it. */
int moeb_set_expert_sources(moeb_stack* s, const void* const* ptrs, size_t n);
/* Diagnostics (MOEB_FFN_TSTAMP=1 at create, batch-1 split-K FFN): device-clock
 * stamps [CTA][8] of the last FFN launch — entry, shared expert issued, certain
 * experts released, certain experts issued, final plan in hand, every row
 * issued, consumers done, end (0: phase not reached). n = words available. */
int moeb_debug_ffn_tstamps(moeb_stack* s, uint64_t* out, size_t cap, size_t* n);
/* MOEB_MODEL_LOG_STEPS: the last prefill's layer `layer`: input hidden
 * (bf16 [N][d]), router scores (fp32 [N][E]), selections in rank order
 * (uint8 [N][k]) and fp32 layer output before the residual ([N][d]); every
 * pointer nullable, n_tokens = N. */
int moeb_get_prefill_log(moeb_stack* s, uint32_t layer, uint32_t* n_tokens, uint16_t* x_in,
                         float* scores, uint8_t* sel, float* y);
/* Synchronise the stack's streams. A device wait that gave up (a lost
 * upload, kSpinLimitNs) is reported here once as status 5 and cleared.
 * Serial mode (MOEB_SERIAL=1, automatic under ncu / nsys / compute-sanitizer):
 * upload dependencies become stream waits set up by the host after each
 * decide kernel instead of in-kernel spins, so tools that serialise kernels
 * see a correct, if slower, pipeline. Steps of different stacks on one
 * device are ordered on the device (the FFN grids need every SM). */
int moeb_sync(moeb_stack* s);

/* Decision counters since create (same vocabulary as Metrics, pipeline.hpp:63-78). */
int moeb_get_metrics(moeb_stack* s, moeb_metrics* m);
/* Per-step decision records (MOEB_MODEL_LOG_STEPS), cumulative since create
 * (first 16384 layer-steps; a longer log returns status 4 rather than a
 * truncated array): JSON array of
 * {"it","layer","mask","tok":[{"sel","sub","kept"}],"load","cpu","pref","evict","completion"}
 * plus the fp32 router scores each step used (for oracle replay). */
int moeb_get_decisions_json(moeb_stack* s, char** json);
int moeb_get_scores(moeb_stack* s, float* out, size_t cap, size_t* n);
/* MOEB_MODEL_PREDICTOR: the predicted fp32 scores each step's prefetch used
 * ([steps][B][E], the step that was the prefetch target; NaN rows: no
 * prediction for that step). */
int moeb_get_pred_scores(moeb_stack* s, float* out, size_t cap, size_t* n);
/* The same per-step records as plain structs (what the C++ MoeStack wrapper,
 * include/moesched/moe_layer.hpp, turns into RouteResult / load-list form).
 * One moeb_step_record per (iteration, layer), batch moeb_token_records each,
 * in step order. Bitmask resident_before = the residency snapshot the router
 * saw (pipeline.cpp:154-155). steps/toks may be NULL to query the count. */
typedef struct moeb_step_record {
  uint64_t iteration;
  uint32_t layer, batch;
  uint64_t resident_before, completion;
  uint8_t n_load, n_cpu, n_pref, n_evict;
  uint8_t load[64], cpu[64], pref[64];     /* load_list, cpu_list (BA-streamed), prefetch issues */
  uint8_t evict_layer[128], evict_expert[128];
} moeb_step_record;
typedef struct moeb_token_record {
  uint8_t n_sel, n_sub, n_kept, pad;
  uint8_t sel[16], sub_dropped[16], sub_chosen[16], kept[16];
} moeb_token_record;
int moeb_get_decisions(moeb_stack* s, moeb_step_record* steps, moeb_token_record* toks, size_t cap_steps,
                       size_t* n_steps);
/* Upload accounting: bytes and the copy stream's busy time (CUDA events). */
typedef struct moeb_io_stats {
  uint64_t h2d_bytes, h2d_copies, d2d_copies, steps;
  double copy_ms; /* copy-stream busy time: one upload in 8 is timed with CUDA events
                   * (MOEB_COPY_TIMING_EVERY=n; 1 = every one) and the sum extrapolated
                   * over all uploads (every upload is one expert) */
  /* speculative uploads (opt-in experiment, MOEB_SPEC_UPLOAD=1; batch-1 stacks
   * with stage Pre and a capped cache): after each decision the first expert of the
   * prefetch queue's ranking that is not resident in the next layer is
   * uploaded into a side buffer in chunks, only while the copy engine has
   * nothing else to do; if the next step uploads that expert anyway it comes
   * from the buffer (promoted: the rest issued at once). Decisions are
   * untouched. h2d_bytes includes the chunks. */
  uint64_t spec_jobs, spec_promoted, spec_chunks, spec_bytes;
} moeb_io_stats;
int moeb_get_io_stats(moeb_stack* s, moeb_io_stats* st);
/* Duration (ms, copy-stream CUDA events) of the timed expert uploads (one in
 * 8 by default, MOEB_COPY_TIMING_EVERY) since create or moeb_reset_kernel_stats
 * (first 65536): per-upload PCIe rates. */
int moeb_get_copy_times(moeb_stack* s, float* ms, size_t cap, size_t* n);
/* Device buffers for tests: fp32 layer outputs of the last step ([L][B][d]) */
int moeb_get_layer_outputs(moeb_stack* s, float* out, size_t cap);
/* Reset the decision state and cache contents to the post-create state
 * (iteration 0), keeping weights and the pinned pool. */
int moeb_reset(moeb_stack* s);
/* The stack's own compute stream (cudaStream_t). */
void* moeb_stream(moeb_stack* s);
/* Per-kernel CUDA-event totals (MOEB_MODEL_TIME_KERNELS) and algorithmic
 * bytes (weights + activations each launch must move at least once). */
typedef struct moeb_kernel_stats {
  double route_ms, ffn_ms;        /* route = fused router gate + decision launch */
  uint64_t route_launches, ffn_launches;
  uint64_t route_bytes, ffn_bytes, ffn_planned;
  uint64_t prof_ns[32];           /* device phase timers of the decision launch (make PROFILE=1) */
} moeb_kernel_stats;
int moeb_get_kernel_stats(moeb_stack* s, moeb_kernel_stats* out);
int moeb_reset_kernel_stats(moeb_stack* s);

/* generate_trace (trace.hpp:45 / trace.cpp:106-151): synthetic skewed gate
 * scores, [iters][L][B][E] fp64 (workload synthesis, host side). */
int moeb_generate_trace(uint32_t L, uint32_t E, uint32_t B, double hot_fraction, double hot_mass,
                        double persistence, double concentration, uint64_t iters, uint64_t seed,
                        double* out);

/* Device-clock (ns) timeline of the last <= 16384 layer-steps, 16 words each:
 * 0 FFN start, 1 FFN saw its last upload land (0: none), 2 FFN end,
 * 3 decide entry, 4 uploads published (mailbox entry A), 5 decide end,
 * 6 FFN has the speculative plan (split-K FFN: the shared expert released
 * right after the gate), 7 FFN CTA 0 entry,
 * 8 tcgen05 FFN: CTA 0 final sum done (other FFN kernels: unused),
 * 9 split-K FFN: the speculative plan of the certain experts, 10 CUDA-core FFN: down pass starts, 11 FFN CTA 0 compute done,
 * 12 final plan released to the FFN, 13 last FFN CTA compute done (max over
 * CTAs), 14 split-K FFN: reduction barrier passed, 15 number of uploads the
 * step published (a count, not a time). Diagnostics only. */
int moeb_get_timeline(moeb_stack* s, uint64_t* out, size_t cap, size_t* n);
/* Pinned host pool pointer and per-expert bytes (for the CPU oracle). */
int moeb_get_host_pool(moeb_stack* s, const void** pool, size_t* expert_bytes);
/* MOEB_MODEL_DOWN_T when the stack's pool is row-interleaved (batch 1),
 * MOEB_MODEL_TILED when it is UMMA-tiled (batched tensor-core FFN). */
int moeb_host_pool_flags(moeb_stack* s, uint32_t* flags);

#ifdef __cplusplus
}
#endif
#endif
