/*
 * cpu_moe.c — TEST / BASELINE INFRASTRUCTURE ONLY.
 *
 * CPU fp32 restatement of the MoE decode layer over bf16 weights in host RAM,
 * threaded over all host cores: the "CPU path" the B200 build is reported
 * beside (the paper's CPU-offload baseline).
 * The reference has no layer arithmetic (it abstracts experts as t_gpu /
 * t_cpu_token tasks, pipeline.cpp:217-259); this follows the semantics in
 * oracle/moe_layer_ref.py. Used only by bench.py's cpu_baseline / --impl
 * reference legs; never linked into the product.
 */
#include <math.h>
#include <pthread.h>
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

typedef struct {
  int kind; /* 0 synth, 1 gemv-gate-up, 2 gemv-down */
  uint64_t seed, tensor, lo, hi;
  float scale;
  uint16_t* out;
  /* gemv */
  const uint16_t* w;
  const float* x;
  float* y;
  uint32_t cols;
} job_t;

static void* run_job(void* p) {
  job_t* j = (job_t*)p;
  if (j->kind == 0) {
    for (uint64_t i = j->lo; i < j->hi; ++i) {
      const uint64_t z = mix64(j->seed ^ (j->tensor * 0x9E3779B97F4A7C15ULL) ^ (i * 0xD1B54A32D192ED03ULL));
      const float u = (float)(uint32_t)(z >> 40) * 5.9604644775390625e-08f;
      j->out[i] = to_bf((2.0f * u - 1.0f) * j->scale);
    }
  } else {
    for (uint64_t r = j->lo; r < j->hi; ++r) {
      const uint16_t* row = j->w + r * j->cols;
      float s = 0.f;
      for (uint32_t c = 0; c < j->cols; ++c) s += bf(row[c]) * j->x[c];
      j->y[r] = s;
    }
  }
  return NULL;
}

static void parallel(job_t* base, int nthreads, uint64_t n) {
  pthread_t th[256];
  job_t jobs[256];
  if (nthreads > 256) nthreads = 256;
  if (nthreads < 1) nthreads = 1;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = *base;
    jobs[t].lo = n * t / nthreads;
    jobs[t].hi = n * (t + 1) / nthreads;
    pthread_create(&th[t], NULL, run_job, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* One tensor of the counter-based weights (weights.cuh), threaded. */
void cpu_synth(uint64_t seed, uint64_t tensor, uint64_t n, uint32_t fan_in, uint16_t* out, int nthreads) {
  job_t j;
  memset(&j, 0, sizeof j);
  j.kind = 0;
  j.seed = seed;
  j.tensor = tensor;
  j.scale = (float)sqrt(3.0 / (double)fan_in);
  j.out = out;
  parallel(&j, nthreads, n);
}

static void gemv(const uint16_t* w, const float* x, float* y, uint64_t rows, uint32_t cols, int nthreads) {
  job_t j;
  memset(&j, 0, sizeof j);
  j.kind = 1;
  j.w = w;
  j.x = x;
  j.y = y;
  j.cols = cols;
  parallel(&j, nthreads, rows);
}

/* SwiGLU expert on one token: w = [gate F*d][up F*d][down d*F]; y += wt * out. */
static void expert(const uint16_t* w, uint32_t d, uint32_t F, const float* u, float wt, float* y,
                   float* scratch, int nthreads) {
  float* g = scratch;
  float* up = scratch + F;
  float* o = scratch + 2 * (size_t)F;
  gemv(w, u, g, F, d, nthreads);
  gemv(w + (size_t)F * d, u, up, F, d, nthreads);
  for (uint32_t i = 0; i < F; ++i) g[i] = g[i] / (1.0f + expf(-g[i])) * up[i];
  gemv(w + 2 * (size_t)F * d, g, o, d, F, nthreads);
  for (uint32_t i = 0; i < d; ++i) y[i] += wt * o[i];
}

/* One MoE layer for one token (B = 1), all in fp32 over bf16 weights:
 * RMSNorm -> router GEMV (logits written out) -> shared expert (optionally
 * sigmoid-gated) + weighted routed experts -> residual. `experts` holds the
 * selected experts' weight pointers, `wts` their combine weights. */
void cpu_moe_layer(const uint16_t* x, uint32_t d, uint32_t F, uint32_t S, uint32_t E,
                   const uint16_t* router, const uint16_t* shared, const uint16_t* shared_gate,
                   const uint16_t* const* experts, const float* wts, uint32_t n_sel, float* logits,
                   float* y, uint16_t* x_next, int nthreads) {
  float* u = (float*)malloc(sizeof(float) * d);
  const uint32_t fmax = F > S ? F : S;
  float* scratch = (float*)malloc(sizeof(float) * (2 * (size_t)fmax + d + 8));
  double ss = 0.0;
  for (uint32_t i = 0; i < d; ++i) ss += (double)bf(x[i]) * bf(x[i]);
  const float inv = (float)(1.0 / sqrt(ss / d + 1e-6));
  for (uint32_t i = 0; i < d; ++i) u[i] = bf(to_bf(bf(x[i]) * inv));
  gemv(router, u, logits, E, d, nthreads);
  memset(y, 0, sizeof(float) * d);
  if (S) {
    float gate = 1.0f;
    if (shared_gate) {
      float z = 0.f;
      for (uint32_t i = 0; i < d; ++i) z += bf(shared_gate[i]) * u[i];
      gate = 1.0f / (1.0f + expf(-z));
    }
    expert(shared, d, S, u, gate, y, scratch, nthreads);
  }
  for (uint32_t i = 0; i < n_sel; ++i) expert(experts[i], d, F, u, wts[i], y, scratch, nthreads);
  for (uint32_t i = 0; i < d; ++i) x_next[i] = to_bf(bf(x[i]) + y[i]);
  free(u);
  free(scratch);
}
