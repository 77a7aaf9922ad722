/*
 * moesched_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C (C11) CPU restatement of the reference decision path
 * (/root/reference/proj/src/{rng,router,cache,prefetch,balancer,pipeline,trace}.cpp)
 * used as the parity checker for the CUDA product path. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * The product library (paper_2508_18983_b200/) never links or calls it.
 *
 * Parity pin: this restatement is checked against (a) the known-answer
 * vectors of the reference's own tests (tests/test_oracle_kats.py) and
 * (b) golden dumps produced by the reference library itself, compiled from
 * /root/reference by oracle/Makefile into oracle/_ref/ (tests/golden/).
 */
#ifndef MOESCHED_ORACLE_H
#define MOESCHED_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_E 256

/* Status codes mirror the product C-ABI (include/moesched_b200.h). */
enum { ORC_OK = 0, ORC_ECONFIG = 1, ORC_EIO = 2, ORC_ECACHE = 3, ORC_ELOGIC = 4 };

typedef struct orc_config {
  uint32_t num_layers, experts, top_k, batch; /* ModelShape core.hpp:40-47 */
  double alpha;                                /* RouterConfig core.hpp:49-51 */
  uint32_t slots, window;                      /* CacheConfig core.hpp:56-61 */
  int32_t policy;                              /* 0 ScoreWindow, 1 LRU */
  int32_t init_fill;                           /* 0 FirstSlots, 1 SeededRandom, 2 Empty */
  uint64_t t_attn, t_gpu, t_cpu_token, t_load, t_route; /* CostModel core.hpp:63-69 */
  double p_top, p_active;                      /* PredictorConfig core.hpp:71-75 */
  uint32_t queue_depth;
  int32_t ce, er, pre, ba;                     /* StageSet core.hpp:82-92 */
  uint64_t seed;
} orc_config;

/* ---- rng (rng.cpp:10-96) ---- */
typedef struct orc_rng { uint64_t s[4]; } orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_u64(orc_rng* r);
double orc_rng_double(orc_rng* r);
uint64_t orc_rng_below(orc_rng* r, uint64_t n);
double orc_rng_normal(orc_rng* r);
double orc_rng_gamma(orc_rng* r, double shape);
uint64_t orc_derive_seed(uint64_t seed, uint64_t tag);

/* ---- router (router.cpp:13-260) ---- */
typedef struct orc_cls {
  double beta, thr_top, thr_low, thr_alt;
  uint32_t n_act, n_top, n_low, n_alt;
  uint32_t act[ORC_MAX_E], top[ORC_MAX_E], low[ORC_MAX_E], alt[ORC_MAX_E];
} orc_cls;

typedef struct orc_token_route {
  uint32_t n_sel, n_sub, n_kept;
  uint32_t sel[ORC_MAX_E];
  uint32_t sub_dropped[ORC_MAX_E], sub_chosen[ORC_MAX_E];
  uint32_t kept[ORC_MAX_E];
  orc_cls cls;
} orc_token_route;

int orc_classify(const double* s, uint32_t E, uint32_t k, double alpha, orc_cls* out);
void orc_plain_top_k(const double* s, uint32_t E, uint32_t k, uint32_t* out, uint32_t* n_out);
/* scores: [B][E]; mask: [E]; toks: [B]; top_set/pending: [E] with counts. */
int orc_route(const double* scores, uint32_t B, uint32_t E, const uint8_t* mask, uint32_t k,
              double alpha, orc_token_route* toks, uint32_t* top_set, uint32_t* n_top_set,
              uint32_t* pending, uint32_t* n_pending);
void orc_coalesce(orc_token_route* toks, const double* scores, uint32_t B, uint32_t E,
                  const uint8_t* mask, const uint32_t* top_set, uint32_t n_top_set,
                  uint32_t* pending, uint32_t* n_pending);

/* ---- balancer (balancer.cpp:8-38) ---- */
void orc_balance(const uint32_t* uid, const uint32_t* batch, uint32_t n, uint64_t t_cpu_token,
                 uint64_t t_load, uint32_t* load_list, uint32_t* n_load, uint32_t* cpu_list,
                 uint32_t* n_cpu, uint64_t* c_load, uint64_t* c_cpu);

/* ---- prefetch (prefetch.cpp:34-115) ---- */
/* head_kind: 0 TopScore, 1 ActiveNonTop, 2 Inactive. supplied may be NULL. */
int orc_predict_scores(const double* true_next, const double* supplied, uint32_t E,
                       double p_top, double p_active, uint32_t k, double alpha, orc_rng* rng,
                       double* out_scores, uint32_t* head, int32_t* head_kind);
void orc_build_queue(const double* predicted, const uint8_t* mask, uint32_t E, uint32_t depth,
                     uint32_t* entries, uint32_t* n_entries);

/* ---- trace (trace.cpp:106-151) ---- */
/* out: [iters][L][B][E] doubles. */
void orc_generate_trace(uint32_t L, uint32_t E, uint32_t B, double hot_fraction,
                        double hot_mass, double persistence, double concentration,
                        uint64_t iters, uint64_t seed, double* out);

/* ---- cache (cache.cpp:10-156) exposed for op-sequence fuzzing ---- */
typedef struct orc_cache orc_cache;
orc_cache* orc_cache_new(uint32_t L, uint32_t E, uint32_t slots, uint32_t window, int32_t policy,
                         int32_t init_fill, uint64_t seed);
void orc_cache_free(orc_cache* c);
uint32_t orc_cache_resident(const orc_cache* c, uint32_t layer, uint32_t* out);
int orc_cache_record(orc_cache* c, uint32_t layer, const double* scores, uint32_t n);
double orc_cache_window_average(const orc_cache* c, uint32_t layer, uint32_t e);
int64_t orc_cache_try_evict(const orc_cache* c, uint32_t layer); /* -1: none */
void orc_cache_shield(orc_cache* c, uint32_t layer, uint32_t e);
void orc_cache_unshield(orc_cache* c, uint32_t layer);
int orc_cache_is_shielded(const orc_cache* c, uint32_t layer, uint32_t e);
void orc_cache_touch(orc_cache* c, uint32_t layer, uint32_t e, uint64_t now);
/* returns ORC_OK/ORC_ECACHE/ORC_ELOGIC; *evicted = -1 when nothing left. */
int orc_cache_admit(orc_cache* c, uint32_t layer, uint32_t e, uint64_t now, int64_t* evicted);

/* ---- pipeline (pipeline.cpp:110-491) ----
 * scores: [iters][L][B][E]; pred: same shape or NULL; has_pred: [iters][L][B] or NULL.
 * Returns a malloc'd JSON document (free with orc_free): {"metrics", "stats",
 * "tasks", "windows", "evictions", "cache_final"[, "steps"]} or {"error": ...}. */
char* orc_simulate_json(const orc_config* cfg, const double* scores, const double* pred,
                        const uint8_t* has_pred, uint64_t iters, int32_t emit_steps,
                        int32_t emit_timeline);
void orc_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
