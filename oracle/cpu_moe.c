/*
 * cpu_moe.c — TEST / BASELINE INFRASTRUCTURE ONLY.
 *
 * CPU fp32 restatement of the MoE decode layer over bf16 weights in host RAM,
 * threaded over all host cores: the "CPU path" the B200 build is reported
 * beside (the paper's CPU-offload baseline).
 * The reference has no layer arithmetic (it abstracts experts as t_gpu /
 * t_cpu_token tasks, pipeline.cpp:217-259); this follows the semantics in
 * oracle/moe_layer_ref.py (pinned to the HF modules by tests/test_hf_pin.py).
 * Used only by bench.py's cpu_baseline / --impl reference legs and the tests;
 * never linked into the product.
 *
 * Built to be a credible CPU baseline, i.e. host-memory-bandwidth bound:
 *   * a persistent worker pool (threads created once, woken through a
 *     generation counter they spin on; no create/join per GEMV);
 *   * two parallel phases per layer: (1) the router rows and every
 *     (gate row r, up row r) pair of the shared and selected experts, split
 *     across threads by rows, each thread forming h_r = silu(g_r . u)(up_r . u)
 *     for its rows directly; (2) the down projections, split by output row,
 *     each thread summing every expert's weighted contribution to its rows;
 *   * AVX2 + FMA bf16 dot products (bf16 -> fp32 is a 16-bit shift, 4
 *     independent 8-wide accumulators), no -ffast-math (the weight generator
 *     below must stay bit-exact with csrc/weights.cuh).
 * cpu_bytes_touched() reports the weight bytes read, so bench.py can state the
 * achieved host GB/s next to the baseline.
 */
#ifndef _POSIX_C_SOURCE
#define _POSIX_C_SOURCE 200809L /* nanosleep */
#endif
#include <immintrin.h>
#include <math.h>
#include <pthread.h>
#include <time.h>
#include <sched.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline float bf(uint16_t b) {
  union { uint32_t u; float f; } v;
  v.u = (uint32_t)b << 16;
  return v.f;
}
static inline uint16_t to_bf(float f) {
  union { uint32_t u; float f; } v;
  v.f = f;
  v.u += 0x7FFFu + ((v.u >> 16) & 1u);
  return (uint16_t)(v.u >> 16);
}
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* ------------------------------------------------------------ worker pool */

typedef void (*task_fn)(void* ctx, int tid, int nthreads);

#define MAX_THREADS 256
static struct {
  int n;                    /* threads including the caller (tid 0) */
  pthread_t th[MAX_THREADS];
  _Atomic uint64_t gen;     /* bumped to start a phase */
  _Atomic int remaining;    /* workers still running the phase */
  task_fn fn;
  void* ctx;
  pthread_mutex_t mu;
} g_pool = {.mu = PTHREAD_MUTEX_INITIALIZER};

static uint64_t g_start_gen[MAX_THREADS];

static void* worker(void* arg) {
  const int tid = (int)(intptr_t)arg;
  uint64_t seen = g_start_gen[tid];  /* the generation current when it was created */
  for (;;) {
    uint64_t g;
    unsigned spins = 0;
    while ((g = atomic_load_explicit(&g_pool.gen, memory_order_acquire)) == seen) {
      /* spin through the short gaps between phases; park once idle (a
       * yielding worker would keep all cores busy and slow the GPU runs'
       * host threads that follow a CPU baseline) */
      if (++spins < (1u << 16)) _mm_pause();
      else {
        struct timespec ts = {0, 100000};
        nanosleep(&ts, NULL);
      }
    }
    seen = g;
    g_pool.fn(g_pool.ctx, tid, g_pool.n);
    atomic_fetch_sub_explicit(&g_pool.remaining, 1, memory_order_acq_rel);
  }
  return NULL;
}

static void pool_ensure(int nthreads) {
  if (nthreads > MAX_THREADS) nthreads = MAX_THREADS;
  if (nthreads < 1) nthreads = 1;
  if (g_pool.n >= nthreads) return;
  if (g_pool.n == 0) g_pool.n = 1;
  for (int t = g_pool.n; t < nthreads; ++t) {
    g_start_gen[t] = atomic_load(&g_pool.gen);
    pthread_create(&g_pool.th[t], NULL, worker, (void*)(intptr_t)t);
    pthread_detach(g_pool.th[t]);
  }
  g_pool.n = nthreads;
}

/* Run fn on every pool thread (the caller is tid 0) and wait for all. */
static void pool_run(task_fn fn, void* ctx) {
  g_pool.fn = fn;
  g_pool.ctx = ctx;
  atomic_store_explicit(&g_pool.remaining, g_pool.n - 1, memory_order_release);
  atomic_fetch_add_explicit(&g_pool.gen, 1, memory_order_acq_rel);
  fn(ctx, 0, g_pool.n);
  while (atomic_load_explicit(&g_pool.remaining, memory_order_acquire) > 0) _mm_pause();
}

static inline void split(uint64_t n, int tid, int nt, uint64_t* lo, uint64_t* hi) {
  *lo = n * (uint64_t)tid / (uint64_t)nt;
  *hi = n * (uint64_t)(tid + 1) / (uint64_t)nt;
}

/* ------------------------------------------------- counter-based weights */

typedef struct {
  uint64_t seed, tensor, n;
  float scale;
  uint16_t* out;
} synth_ctx;

static void synth_task(void* p, int tid, int nt) {
  const synth_ctx* c = (const synth_ctx*)p;
  uint64_t lo, hi;
  split(c->n, tid, nt, &lo, &hi);
  for (uint64_t i = lo; i < hi; ++i) {
    const uint64_t z = mix64(c->seed ^ (c->tensor * 0x9E3779B97F4A7C15ULL) ^ (i * 0xD1B54A32D192ED03ULL));
    const float u = (float)(uint32_t)(z >> 40) * 5.9604644775390625e-08f;
    const float w = 2.0f * u - 1.0f;
    c->out[i] = to_bf(w * c->scale);
  }
}

/* One tensor of the counter-based weights (weights.cuh), threaded. */
void cpu_synth(uint64_t seed, uint64_t tensor, uint64_t n, uint32_t fan_in, uint16_t* out, int nthreads) {
  pthread_mutex_lock(&g_pool.mu);
  pool_ensure(nthreads);
  synth_ctx c = {seed, tensor, n, (float)sqrt(3.0 / (double)fan_in), out};
  pool_run(synth_task, &c);
  pthread_mutex_unlock(&g_pool.mu);
}

/* ------------------------------------------------------------ bf16 dots */

static inline __m256 bf8(const uint16_t* p) {
  const __m128i h = _mm_loadu_si128((const __m128i*)p);
  return _mm256_castsi256_ps(_mm256_slli_epi32(_mm256_cvtepu16_epi32(h), 16));
}

static inline float hsum(__m256 v) {
  __m128 s = _mm_add_ps(_mm256_castps256_ps128(v), _mm256_extractf128_ps(v, 1));
  s = _mm_add_ps(s, _mm_movehl_ps(s, s));
  s = _mm_add_ss(s, _mm_shuffle_ps(s, s, 1));
  return _mm_cvtss_f32(s);
}

/* dot(bf16 row[n], fp32 x[n]); n a multiple of 8 */
static inline float dot_bf16(const uint16_t* w, const float* x, uint32_t n) {
  __m256 a0 = _mm256_setzero_ps(), a1 = a0, a2 = a0, a3 = a0;
  uint32_t i = 0;
  for (; i + 32 <= n; i += 32) {
    a0 = _mm256_fmadd_ps(bf8(w + i), _mm256_loadu_ps(x + i), a0);
    a1 = _mm256_fmadd_ps(bf8(w + i + 8), _mm256_loadu_ps(x + i + 8), a1);
    a2 = _mm256_fmadd_ps(bf8(w + i + 16), _mm256_loadu_ps(x + i + 16), a2);
    a3 = _mm256_fmadd_ps(bf8(w + i + 24), _mm256_loadu_ps(x + i + 24), a3);
  }
  for (; i + 8 <= n; i += 8) a0 = _mm256_fmadd_ps(bf8(w + i), _mm256_loadu_ps(x + i), a0);
  float s = hsum(_mm256_add_ps(_mm256_add_ps(a0, a1), _mm256_add_ps(a2, a3)));
  for (; i < n; ++i) s += bf(w[i]) * x[i];
  return s;
}

/* ------------------------------------------------------------- the layer */

#define MAX_ITEMS 80
typedef struct {
  const uint16_t* w;  /* [gate F*d][up F*d][down d*F] */
  uint32_t F;
  float wt;
  float* h;           /* [F] intermediate activations */
  uint64_t row0;      /* first global row of this item in phase 1 */
} item_t;

typedef struct {
  uint32_t d, E, n_items;
  const uint16_t* router;
  const float* u;
  float* logits;
  item_t it[MAX_ITEMS];
  uint64_t rows1;     /* E + sum F */
  float* y;
} layer_ctx;

static void phase1(void* p, int tid, int nt) {
  layer_ctx* c = (layer_ctx*)p;
  uint64_t lo, hi;
  split(c->rows1, tid, nt, &lo, &hi);
  const uint32_t d = c->d;
  for (uint64_t r = lo; r < hi;) {
    if (r < c->E) {  /* router rows */
      c->logits[r] = dot_bf16(c->router + r * d, c->u, d);
      ++r;
      continue;
    }
    uint32_t k = 0;
    while (k + 1 < c->n_items && c->it[k + 1].row0 <= r) ++k;
    item_t* t = &c->it[k];
    const uint64_t end = t->row0 + t->F < hi ? t->row0 + t->F : hi;
    const uint16_t* g = t->w;
    const uint16_t* up = t->w + (size_t)t->F * d;
    for (; r < end; ++r) {
      const uint64_t j = r - t->row0;
      const float gv = dot_bf16(g + j * d, c->u, d);
      const float uv = dot_bf16(up + j * d, c->u, d);
      t->h[j] = gv / (1.0f + expf(-gv)) * uv;
    }
  }
}

static void phase2(void* p, int tid, int nt) {
  layer_ctx* c = (layer_ctx*)p;
  uint64_t lo, hi;
  split(c->d, tid, nt, &lo, &hi);
  const uint32_t d = c->d;
  for (uint64_t i = lo; i < hi; ++i) {
    float s = 0.f;
    for (uint32_t k = 0; k < c->n_items; ++k) {
      const item_t* t = &c->it[k];
      const uint16_t* dn = t->w + 2 * (size_t)t->F * d;
      s += t->wt * dot_bf16(dn + i * t->F, t->h, t->F);
    }
    c->y[i] = s;
  }
}

static _Atomic uint64_t g_bytes;

/* One MoE layer for one token (B = 1), all in fp32 over bf16 weights:
 * RMSNorm -> router GEMV (logits written out) -> shared expert (optionally
 * sigmoid-gated) + weighted routed experts -> residual. `experts` holds the
 * selected experts' weight pointers, `wts` their combine weights. */
void cpu_moe_layer(const uint16_t* x, uint32_t d, uint32_t F, uint32_t S, uint32_t E,
                   const uint16_t* router, const uint16_t* shared, const uint16_t* shared_gate,
                   const uint16_t* const* experts, const float* wts, uint32_t n_sel, float* logits,
                   float* y, uint16_t* x_next, int nthreads) {
  pthread_mutex_lock(&g_pool.mu);
  pool_ensure(nthreads);
  static layer_ctx c;  /* under g_pool.mu */
  float* u = (float*)aligned_alloc(64, sizeof(float) * ((d + 15) & ~15u));
  const uint32_t n_items = (S ? 1 : 0) + n_sel;
  float* hbuf = (float*)malloc(sizeof(float) * ((size_t)S + (size_t)n_sel * F + 8));
  double ss = 0.0;
  for (uint32_t i = 0; i < d; ++i) ss += (double)bf(x[i]) * bf(x[i]);
  const float inv = (float)(1.0 / sqrt(ss / d + 1e-6));
  for (uint32_t i = 0; i < d; ++i) u[i] = bf(to_bf(bf(x[i]) * inv));
  float gate = 1.0f;
  if (S && shared_gate) {
    const float z = dot_bf16(shared_gate, u, d);
    gate = 1.0f / (1.0f + expf(-z));
  }
  c.d = d;
  c.E = E;
  c.router = router;
  c.u = u;
  c.logits = logits;
  c.y = y;
  c.n_items = n_items > MAX_ITEMS ? MAX_ITEMS : n_items;
  uint64_t row = E, hoff = 0, bytes = (uint64_t)E * d * 2;
  for (uint32_t k = 0; k < c.n_items; ++k) {
    item_t* t = &c.it[k];
    const int sh = S && k == 0;
    t->w = sh ? shared : experts[k - (S ? 1 : 0)];
    t->F = sh ? S : F;
    t->wt = sh ? gate : wts[k - (S ? 1 : 0)];
    t->h = hbuf + hoff;
    t->row0 = row;
    row += t->F;
    hoff += t->F;
    bytes += 3ull * t->F * d * 2;
  }
  c.rows1 = row;
  pool_run(phase1, &c);
  pool_run(phase2, &c);
  for (uint32_t i = 0; i < d; ++i) x_next[i] = to_bf(bf(x[i]) + y[i]);
  atomic_fetch_add(&g_bytes, bytes);
  pthread_mutex_unlock(&g_pool.mu);
  free(u);
  free(hbuf);
}

/* Weight bytes read by cpu_moe_layer since the last call (then reset). */
uint64_t cpu_bytes_touched(void) { return atomic_exchange(&g_bytes, 0); }

/* ------------------------------------------------------------ prefill */
/* The prefill layer (csrc/prefill.cuh restated on the CPU): N tokens, plain
 * top-k routing (score desc, index asc: router.cpp:252-260), the shared
 * expert + the selected experts batched per expert: every weight row is read
 * once per layer and reused across all of that expert's tokens (phase 1 by
 * (item, intermediate row), phase 2 by output row). */
#define PF_MAX_ITEMS 80
typedef struct {
  const uint16_t* w;
  uint32_t F, n;        /* intermediate rows, tokens */
  const uint32_t* tok;  /* [n] */
  const float* wt;      /* [n] */
  float* h;             /* [n][F] */
  uint64_t row0;        /* first phase-1 row */
} pf_item;

typedef struct {
  uint32_t N, d, E, k, n_items;
  const uint16_t* router;
  const uint16_t* shared_gate;
  float* u;             /* [N][d] */
  float* logits;        /* [N][E] */
  float* sg;            /* [N] */
  pf_item it[PF_MAX_ITEMS];
  uint64_t rows1;
  float* y;             /* [N][d] */
} pf_ctx;

static void pf_route(void* p, int tid, int nt) {
  pf_ctx* c = (pf_ctx*)p;
  uint64_t lo, hi;
  split(c->N, tid, nt, &lo, &hi);
  for (uint64_t t = lo; t < hi; ++t) {
    const float* u = c->u + t * c->d;
    for (uint32_t e = 0; e < c->E; ++e) c->logits[t * c->E + e] = dot_bf16(c->router + (size_t)e * c->d, u, c->d);
    c->sg[t] = c->shared_gate ? 1.0f / (1.0f + expf(-dot_bf16(c->shared_gate, u, c->d))) : 1.0f;
  }
}

static void pf_phase1(void* p, int tid, int nt) {
  pf_ctx* c = (pf_ctx*)p;
  uint64_t lo, hi;
  split(c->rows1, tid, nt, &lo, &hi);
  const uint32_t d = c->d;
  for (uint64_t r = lo; r < hi;) {
    uint32_t k = 0;
    while (k + 1 < c->n_items && c->it[k + 1].row0 <= r) ++k;
    pf_item* t = &c->it[k];
    const uint64_t end = t->row0 + t->F < hi ? t->row0 + t->F : hi;
    for (; r < end; ++r) {
      const uint64_t j = r - t->row0;
      const uint16_t* g = t->w + j * d;
      const uint16_t* up = t->w + (size_t)t->F * d + j * d;
      for (uint32_t i = 0; i < t->n; ++i) {
        const float* u = c->u + (size_t)t->tok[i] * d;
        const float gv = dot_bf16(g, u, d), uv = dot_bf16(up, u, d);
        t->h[(size_t)i * t->F + j] = gv / (1.0f + expf(-gv)) * uv;
      }
    }
  }
}

static void pf_phase2(void* p, int tid, int nt) {
  pf_ctx* c = (pf_ctx*)p;
  uint64_t lo, hi;
  split(c->d, tid, nt, &lo, &hi);
  const uint32_t d = c->d;
  for (uint64_t o = lo; o < hi; ++o)
    for (uint32_t k = 0; k < c->n_items; ++k) {
      const pf_item* t = &c->it[k];
      const uint16_t* dn = t->w + 2 * (size_t)t->F * d + o * t->F;
      for (uint32_t i = 0; i < t->n; ++i)
        c->y[(size_t)t->tok[i] * d + o] += t->wt[i] * dot_bf16(dn, t->h + (size_t)i * t->F, t->F);
    }
}

/* x, x_next: [N][d] bf16; experts: [E] weight pointers ([gate][up][down]);
 * y_out (nullable): the fp32 layer output [N][d]. */
void cpu_moe_prefill_layer(const uint16_t* x, uint32_t N, uint32_t d, uint32_t F, uint32_t S, uint32_t E,
                           uint32_t k, const uint16_t* router, const uint16_t* shared,
                           const uint16_t* shared_gate, const uint16_t* const* experts, int renormalize,
                           float routed_scale, uint16_t* x_next, float* y_out, int nthreads) {
  pthread_mutex_lock(&g_pool.mu);
  pool_ensure(nthreads);
  static pf_ctx c;  /* under g_pool.mu */
  c.N = N;
  c.d = d;
  c.E = E;
  c.k = k;
  c.router = router;
  c.shared_gate = S ? shared_gate : NULL;
  c.u = (float*)aligned_alloc(64, sizeof(float) * (size_t)N * d);
  c.logits = (float*)malloc(sizeof(float) * (size_t)N * E);
  c.sg = (float*)malloc(sizeof(float) * N);
  c.y = (float*)calloc((size_t)N * d, sizeof(float));
  for (uint32_t t = 0; t < N; ++t) {
    const uint16_t* xt = x + (size_t)t * d;
    double ss = 0.0;
    for (uint32_t i = 0; i < d; ++i) ss += (double)bf(xt[i]) * bf(xt[i]);
    const float inv = (float)(1.0 / sqrt(ss / d + 1e-6));
    for (uint32_t i = 0; i < d; ++i) c.u[(size_t)t * d + i] = bf(to_bf(bf(xt[i]) * inv));
  }
  pool_run(pf_route, &c);
  /* softmax, plain top-k, combine weights; per-expert token lists */
  uint32_t* cnt = (uint32_t*)calloc(E, sizeof(uint32_t));
  uint32_t* sel = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)N * k);
  float* wsel = (float*)malloc(sizeof(float) * (size_t)N * k);
  float* sc = (float*)malloc(sizeof(float) * E);
  for (uint32_t t = 0; t < N; ++t) {
    const float* lg = c.logits + (size_t)t * E;
    float m = lg[0];
    for (uint32_t e = 1; e < E; ++e) m = lg[e] > m ? lg[e] : m;
    float s = 0.f;
    for (uint32_t e = 0; e < E; ++e) s += (sc[e] = expf(lg[e] - m));
    for (uint32_t e = 0; e < E; ++e) sc[e] /= s;
    float den = 0.f;
    for (uint32_t e = 0; e < E; ++e) {
      uint32_t rk = 0;
      for (uint32_t j = 0; j < E; ++j) rk += (sc[j] > sc[e] || (sc[j] == sc[e] && j < e));
      if (rk < k) {
        sel[(size_t)t * k + rk] = e;
        wsel[(size_t)t * k + rk] = sc[e];
      }
    }
    for (uint32_t r = 0; r < k; ++r) den += wsel[(size_t)t * k + r];
    for (uint32_t r = 0; r < k; ++r) {
      float w = wsel[(size_t)t * k + r];
      if (renormalize) w /= den;
      wsel[(size_t)t * k + r] = w * routed_scale;
      ++cnt[sel[(size_t)t * k + r]];
    }
  }
  uint32_t* toks = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)N * k + N));
  float* tw = (float*)malloc(sizeof(float) * ((size_t)N * k + N));
  uint64_t hsz = (uint64_t)N * S;
  for (uint32_t e = 0; e < E; ++e) hsz += (uint64_t)cnt[e] * F;
  float* hbuf = (float*)malloc(sizeof(float) * (hsz + 8));
  uint32_t n_items = 0, off = 0;
  uint64_t row = 0, hoff = 0;
  if (S) {
    pf_item* it = &c.it[n_items++];
    it->w = shared;
    it->F = S;
    it->n = N;
    for (uint32_t t = 0; t < N; ++t) {
      toks[t] = t;
      tw[t] = c.sg[t];
    }
    it->tok = toks;
    it->wt = tw;
    off = N;
  }
  for (uint32_t e = 0; e < E; ++e) {
    if (!cnt[e]) continue;
    pf_item* it = &c.it[n_items++];
    it->w = experts[e];
    it->F = F;
    it->n = 0;
    it->tok = toks + off;
    it->wt = tw + off;
    for (uint32_t t = 0; t < N; ++t)
      for (uint32_t r = 0; r < k; ++r)
        if (sel[(size_t)t * k + r] == e) {
          toks[off + it->n] = t;
          tw[off + it->n] = wsel[(size_t)t * k + r];
          ++it->n;
        }
    off += it->n;
  }
  for (uint32_t i = 0; i < n_items; ++i) {
    c.it[i].row0 = row;
    c.it[i].h = hbuf + hoff;
    row += c.it[i].F;
    hoff += (uint64_t)c.it[i].n * c.it[i].F;
    atomic_fetch_add(&g_bytes, 3ull * c.it[i].F * d * 2);
  }
  c.n_items = n_items;
  c.rows1 = row;
  pool_run(pf_phase1, &c);
  pool_run(pf_phase2, &c);
  for (size_t i = 0; i < (size_t)N * d; ++i) x_next[i] = to_bf(bf(x[i]) + c.y[i]);
  if (y_out) memcpy(y_out, c.y, sizeof(float) * (size_t)N * d);
  pthread_mutex_unlock(&g_pool.mu);
  free(c.u);
  free(c.logits);
  free(c.sg);
  free(c.y);
  free(cnt);
  free(sel);
  free(wsel);
  free(sc);
  free(toks);
  free(tw);
  free(hbuf);
}
