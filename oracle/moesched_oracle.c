/*
 * moesched_oracle.c — TEST INFRASTRUCTURE ONLY (see moesched_oracle.h).
 *
 * Plain-C restatement of the reference decision path. Every function cites
 * the reference file:line it restates (paths relative to
 * /root/reference/proj/src). This file is the checker the CUDA product is
 * compared against; it is never linked into the product library.
 */
#include "moesched_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */
/* rng.cpp:12-18 splitmix64 */
static uint64_t sm64(uint64_t* s) {
  *s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.cpp:26-31 */
void orc_rng_seed(orc_rng* r, uint64_t seed) {
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = sm64(&s);
}
/* rng.cpp:33-43 xoshiro256** */
uint64_t orc_rng_u64(orc_rng* r) {
  uint64_t* s = r->s;
  const uint64_t out = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return out;
}
/* rng.cpp:45-47 */
double orc_rng_double(orc_rng* r) { return (double)(orc_rng_u64(r) >> 11) * 0x1.0p-53; }
/* rng.cpp:49-56 */
uint64_t orc_rng_below(orc_rng* r, uint64_t n) {
  const uint64_t lim = n * (UINT64_MAX / n);
  uint64_t x;
  do { x = orc_rng_u64(r); } while (x >= lim);
  return x % n;
}
/* rng.cpp:58-64 */
double orc_rng_normal(orc_rng* r) {
  const double u1 = 1.0 - orc_rng_double(r);
  const double u2 = orc_rng_double(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}
/* rng.cpp:66-89 Marsaglia-Tsang */
double orc_rng_gamma(orc_rng* r, double shape) {
  if (shape < 1.0) {
    const double u = 1.0 - orc_rng_double(r);
    return orc_rng_gamma(r, shape + 1.0) * pow(u, 1.0 / shape);
  }
  const double d = shape - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    const double x = orc_rng_normal(r);
    const double t = 1.0 + c * x;
    if (t <= 0.0) continue;
    const double v = t * t * t;
    const double u = orc_rng_double(r);
    if (u < 1.0 - 0.0331 * x * x * x * x) return d * v;
    if (u > 0.0 && log(u) < 0.5 * x * x + d * (1.0 - v + log(v))) return d * v;
  }
}
/* rng.cpp:91-96 */
uint64_t orc_derive_seed(uint64_t seed, uint64_t tag) {
  uint64_t s = seed ^ (0x6a09e667f3bcc909ULL + tag);
  const uint64_t a = sm64(&s);
  const uint64_t b = sm64(&s);
  return a ^ rotl64(b, 29);
}

/* --------------------------------------------------------------- router */
/* Canonical order: score descending, index ascending (router.cpp:13-25).
 * Insertion sort: E <= 256, and the order is total so any sort agrees. */
static void rank_order(const double* s, uint32_t E, uint32_t* order) {
  for (uint32_t i = 0; i < E; ++i) {
    uint32_t j = i;
    while (j > 0) {
      const uint32_t p = order[j - 1];
      const int before = (s[i] > s[p]) || (s[i] == s[p] && i < p);
      if (!before) break;
      order[j] = p;
      --j;
    }
    order[j] = i;
  }
}

/* router.cpp:35-39 */
void orc_plain_top_k(const double* s, uint32_t E, uint32_t k, uint32_t* out, uint32_t* n_out) {
  uint32_t order[ORC_MAX_E];
  rank_order(s, E, order);
  const uint32_t n = k < E ? k : E;
  memcpy(out, order, n * sizeof(uint32_t));
  *n_out = n;
}

/* router.cpp:41-71 */
int orc_classify(const double* s, uint32_t E, uint32_t k, double alpha, orc_cls* c) {
  if (E <= k) return ORC_ECONFIG;
  uint32_t order[ORC_MAX_E];
  rank_order(s, E, order);
  c->beta = s[order[k]];
  c->thr_top = (1.0 + alpha) * c->beta;
  c->thr_low = c->beta;
  c->thr_alt = (1.0 - alpha) * c->beta;
  c->n_act = k;
  c->n_top = c->n_low = c->n_alt = 0;
  for (uint32_t i = 0; i < k; ++i) {
    const uint32_t e = order[i];
    c->act[i] = e;
    const int low = c->beta > 0.0 && s[e] >= c->thr_low && s[e] < c->thr_top;
    if (low) c->low[c->n_low++] = e;
    else c->top[c->n_top++] = e;
  }
  for (uint32_t i = k; i < E; ++i) {
    const uint32_t e = order[i];
    if (c->beta > 0.0 && s[e] >= c->thr_alt && s[e] < c->thr_low) c->alt[c->n_alt++] = e;
  }
  return ORC_OK;
}

static void sort_u32(uint32_t* v, uint32_t n) {
  for (uint32_t i = 1; i < n; ++i) {
    uint32_t x = v[i], j = i;
    while (j > 0 && v[j - 1] > x) { v[j] = v[j - 1]; --j; }
    v[j] = x;
  }
}
static uint32_t sort_unique_u32(uint32_t* v, uint32_t n) {
  sort_u32(v, n);
  uint32_t m = 0;
  for (uint32_t i = 0; i < n; ++i)
    if (m == 0 || v[m - 1] != v[i]) v[m++] = v[i];
  return m;
}

/* router.cpp:97-152 (Algorithm 1, two passes) */
int orc_route(const double* scores, uint32_t B, uint32_t E, const uint8_t* mask, uint32_t k,
              double alpha, orc_token_route* toks, uint32_t* top_set, uint32_t* n_top_set,
              uint32_t* pending, uint32_t* n_pending) {
  uint8_t inC[ORC_MAX_E];
  memset(inC, 0, sizeof inC);
  for (uint32_t t = 0; t < B; ++t) {
    orc_token_route* tk = &toks[t];
    int rc = orc_classify(scores + (size_t)t * E, E, k, alpha, &tk->cls);
    if (rc) return rc;
    tk->n_sel = tk->n_sub = tk->n_kept = 0;
    for (uint32_t i = 0; i < tk->cls.n_top; ++i) {
      tk->sel[tk->n_sel++] = tk->cls.top[i];
      inC[tk->cls.top[i]] = 1;
    }
  }
  uint32_t nc = 0;
  for (uint32_t e = 0; e < E; ++e)
    if (inC[e]) top_set[nc++] = e;
  *n_top_set = nc;

  uint32_t pend[ORC_MAX_E * 8];
  uint32_t np = 0;
  for (uint32_t t = 0; t < B; ++t) {
    orc_token_route* tk = &toks[t];
    uint32_t blow[ORC_MAX_E], nb = 0, alt[ORC_MAX_E], na = 0;
    for (uint32_t i = 0; i < tk->cls.n_low; ++i) {
      const uint32_t e = tk->cls.low[i];
      if (mask[e] || inC[e]) tk->sel[tk->n_sel++] = e;
      else blow[nb++] = e;
    }
    for (uint32_t i = 0; i < tk->cls.n_alt; ++i) {
      const uint32_t e = tk->cls.alt[i];
      if (mask[e] || inC[e]) alt[na++] = e;
    }
    const uint32_t covered = nb < na ? nb : na;
    const uint32_t kept = nb - covered;
    for (uint32_t i = 0; i < kept; ++i) {
      tk->sel[tk->n_sel++] = blow[i];
      tk->kept[tk->n_kept++] = blow[i];
      if (np < ORC_MAX_E * 8) pend[np++] = blow[i];
    }
    for (uint32_t i = 0; i < covered; ++i) {
      tk->sel[tk->n_sel++] = alt[i];
      tk->sub_dropped[tk->n_sub] = blow[kept + i];
      tk->sub_chosen[tk->n_sub] = alt[i];
      tk->n_sub++;
    }
  }
  np = sort_unique_u32(pend, np);
  memcpy(pending, pend, np * sizeof(uint32_t));
  *n_pending = np;
  return ORC_OK;
}

/* router.cpp:154-260 (fixed-point batch coalescing) */
void orc_coalesce(orc_token_route* toks, const double* scores, uint32_t B, uint32_t E,
                  const uint8_t* mask, const uint32_t* top_set, uint32_t n_top_set,
                  uint32_t* pending, uint32_t* n_pending) {
  if (B == 0) { *n_pending = 0; return; }
  uint32_t cnt[ORC_MAX_E];
  uint8_t inC[ORC_MAX_E];
  memset(cnt, 0, sizeof cnt);
  memset(inC, 0, sizeof inC);
  for (uint32_t t = 0; t < B; ++t)
    for (uint32_t i = 0; i < toks[t].n_sel; ++i) cnt[toks[t].sel[i]]++;
  for (uint32_t i = 0; i < n_top_set; ++i) inC[top_set[i]] = 1;

  int changed = 1;
  while (changed) {
    changed = 0;
    for (uint32_t t = 0; t < B; ++t) {
      orc_token_route* tk = &toks[t];
      const double* s = scores + (size_t)t * E;
      uint8_t sel[ORC_MAX_E], act[ORC_MAX_E];
      memset(sel, 0, E);
      memset(act, 0, E);
      for (uint32_t i = 0; i < tk->n_sel; ++i) sel[tk->sel[i]] = 1;
      for (uint32_t i = 0; i < tk->cls.n_act; ++i) act[tk->cls.act[i]] = 1;

      for (uint32_t li = 0; li < tk->cls.n_low; ++li) {
        const uint32_t orig = tk->cls.low[li];
        uint32_t occupant;
        int sub_idx = -1;
        int is_kept = 0;
        for (uint32_t i = 0; i < tk->n_kept; ++i)
          if (tk->kept[i] == orig) { is_kept = 1; break; }
        if (is_kept) {
          occupant = orig;
        } else {
          for (uint32_t i = 0; i < tk->n_sub; ++i)
            if (tk->sub_dropped[i] == orig) { sub_idx = (int)i; break; }
          if (sub_idx < 0) continue;
          occupant = tk->sub_chosen[sub_idx];
        }
        const uint32_t occ_others = cnt[occupant] - 1;
        uint32_t best = occupant, best_others = occ_others;
        for (uint32_t x = 0; x < E; ++x) {
          const double sx = s[x];
          if (!(tk->cls.beta > 0.0 && sx >= tk->cls.thr_alt && sx < tk->cls.thr_low)) continue;
          if (act[x] || sel[x]) continue;
          const uint32_t others = cnt[x];
          if (!(mask[x] || inC[x] || others > 0)) continue;
          if (others > best_others ||
              (others == best_others && best != occupant &&
               (sx > s[best] || (sx == s[best] && x < best)))) {
            best = x;
            best_others = others;
          }
        }
        if (best == occupant || best_others <= occ_others) continue;
        for (uint32_t i = 0; i < tk->n_sel; ++i)
          if (tk->sel[i] == occupant) { tk->sel[i] = best; break; }
        sel[occupant] = 0;
        sel[best] = 1;
        cnt[occupant]--;
        cnt[best]++;
        if (sub_idx >= 0) {
          tk->sub_chosen[sub_idx] = best;
        } else {
          uint32_t w = 0;
          int erased = 0;
          for (uint32_t i = 0; i < tk->n_kept; ++i) {
            if (!erased && tk->kept[i] == orig) { erased = 1; continue; }
            tk->kept[w++] = tk->kept[i];
          }
          tk->n_kept = w;
          tk->sub_dropped[tk->n_sub] = orig;
          tk->sub_chosen[tk->n_sub] = best;
          tk->n_sub++;
        }
        changed = 1;
      }
    }
  }
  uint32_t pend[ORC_MAX_E * 8], np = 0;
  for (uint32_t t = 0; t < B; ++t)
    for (uint32_t i = 0; i < toks[t].n_kept; ++i)
      if (!mask[toks[t].kept[i]] && np < ORC_MAX_E * 8) pend[np++] = toks[t].kept[i];
  np = sort_unique_u32(pend, np);
  memcpy(pending, pend, np * sizeof(uint32_t));
  *n_pending = np;
}

/* ------------------------------------------------------------- balancer */
/* balancer.cpp:8-38 */
void orc_balance(const uint32_t* uid, const uint32_t* batch, uint32_t n, uint64_t t_cpu_token,
                 uint64_t t_load, uint32_t* load_list, uint32_t* n_load, uint32_t* cpu_list,
                 uint32_t* n_cpu, uint64_t* c_load, uint64_t* c_cpu) {
  uint32_t idx[ORC_MAX_E * 8];
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t j = i;
    while (j > 0) {
      const uint32_t p = idx[j - 1];
      const int before = batch[i] > batch[p] || (batch[i] == batch[p] && uid[i] < uid[p]);
      if (!before) break;
      idx[j] = p;
      --j;
    }
    idx[j] = i;
  }
  *n_load = *n_cpu = 0;
  *c_load = *c_cpu = 0;
  if (n == 0) return;
  size_t l = 0, r = n - 1;
  while (l <= r) {
    if (*c_load <= *c_cpu) {
      *c_load += t_load;
      load_list[(*n_load)++] = uid[idx[l]];
      ++l;
    } else {
      *c_cpu += (uint64_t)batch[idx[r]] * t_cpu_token;
      cpu_list[(*n_cpu)++] = uid[idx[r]];
      if (r == 0) break;
      --r;
    }
  }
}

/* ------------------------------------------------------------- prefetch */
/* prefetch.cpp:12-20 */
static uint32_t argmax_first(const double* s, uint32_t E) {
  uint32_t b = 0;
  for (uint32_t i = 1; i < E; ++i)
    if (s[i] > s[b]) b = i;
  return b;
}
static int in_list(const uint32_t* v, uint32_t n, uint32_t x) {
  for (uint32_t i = 0; i < n; ++i)
    if (v[i] == x) return 1;
  return 0;
}
/* prefetch.cpp:22-32 */
static int32_t head_kind_of(uint32_t head, const orc_cls* c) {
  if (in_list(c->top, c->n_top, head)) return 0;
  if (in_list(c->act, c->n_act, head)) return 1;
  return 2;
}
/* prefetch.cpp:34-83 */
int orc_predict_scores(const double* tn, const double* supplied, uint32_t E, double p_top,
                       double p_active, uint32_t k, double alpha, orc_rng* rng, double* out,
                       uint32_t* head, int32_t* head_kind) {
  orc_cls c;
  int rc = orc_classify(tn, E, k, alpha, &c);
  if (rc) return rc;
  if (supplied) {
    memcpy(out, supplied, E * sizeof(double));
    *head = argmax_first(out, E);
    *head_kind = head_kind_of(*head, &c);
    return ORC_OK;
  }
  uint32_t h;
  if (orc_rng_double(rng) < p_top && c.n_top > 0) {
    h = c.top[orc_rng_below(rng, c.n_top)];
    *head_kind = 0;
  } else {
    uint32_t lows[ORC_MAX_E], nl = 0, ina[ORC_MAX_E], ni = 0;
    for (uint32_t i = 0; i < c.n_act; ++i)
      if (!in_list(c.top, c.n_top, c.act[i])) lows[nl++] = c.act[i];
    for (uint32_t e = 0; e < E; ++e)
      if (!in_list(c.act, c.n_act, e)) ina[ni++] = e;
    if (orc_rng_double(rng) < p_active && nl > 0) {
      h = lows[orc_rng_below(rng, nl)];
      *head_kind = 1;
    } else {
      h = ina[orc_rng_below(rng, ni)];
      *head_kind = 2;
    }
  }
  memcpy(out, tn, E * sizeof(double));
  const uint32_t tt = argmax_first(tn, E);
  const double tmp = out[h];
  out[h] = out[tt];
  out[tt] = tmp;
  *head = h;
  return ORC_OK;
}
/* prefetch.cpp:85-115 */
void orc_build_queue(const double* pred, const uint8_t* mask, uint32_t E, uint32_t depth,
                     uint32_t* entries, uint32_t* n_entries) {
  *n_entries = 0;
  if (depth == 0) return;
  uint32_t order[ORC_MAX_E];
  rank_order(pred, E, order);
  for (uint32_t i = 0; i < E && *n_entries < depth; ++i)
    if (!mask[order[i]]) entries[(*n_entries)++] = order[i];
}

/* ---------------------------------------------------------------- trace */
/* trace.cpp:26-51 */
static void evolve_hot(uint32_t* hot, uint32_t h, uint32_t E, double persistence, orc_rng* rng) {
  uint8_t in_new[ORC_MAX_E];
  memset(in_new, 0, sizeof in_new);
  uint32_t kept[ORC_MAX_E], nk = 0;
  for (uint32_t i = 0; i < h; ++i)
    if (orc_rng_double(rng) < persistence) { kept[nk++] = hot[i]; in_new[hot[i]] = 1; }
  const uint32_t need = h - nk;
  for (uint32_t i = 0; i < need; ++i) {
    uint32_t cand[ORC_MAX_E], nc = 0;
    for (uint32_t e = 0; e < E; ++e)
      if (!in_new[e]) cand[nc++] = e;
    const uint32_t pick = cand[orc_rng_below(rng, nc)];
    kept[nk++] = pick;
    in_new[pick] = 1;
  }
  sort_u32(kept, nk);
  memcpy(hot, kept, nk * sizeof(uint32_t));
}

/* trace.cpp:106-151 (+ helpers :62-102) */
void orc_generate_trace(uint32_t L, uint32_t E, uint32_t B, double hot_fraction, double hot_mass,
                        double persistence, double concentration, uint64_t iters, uint64_t seed,
                        double* out) {
  orc_rng rng;
  orc_rng_seed(&rng, orc_derive_seed(seed, 0x7ace5eedULL));
  long hr = lround(hot_fraction * (double)E);
  uint32_t h = (uint32_t)hr; /* static_cast<uint32_t>(lround(...)) then clamp [1, E] */
  if (h < 1) h = 1;
  if (h > E) h = E;
  uint32_t* hot = (uint32_t*)malloc((size_t)L * ORC_MAX_E * sizeof(uint32_t));
  for (uint32_t l = 0; l < L; ++l) {
    uint32_t pool[ORC_MAX_E];
    for (uint32_t i = 0; i < E; ++i) pool[i] = i;
    uint32_t* hl = hot + (size_t)l * ORC_MAX_E;
    for (uint32_t i = 0; i < h; ++i) {
      const uint64_t j = i + orc_rng_below(&rng, E - i);
      const uint32_t tmp = pool[i];
      pool[i] = pool[j];
      pool[j] = tmp;
      hl[i] = pool[i];
    }
    sort_u32(hl, h);
  }
  const double hot_shape = 1.0 / (concentration > 1e-9 ? concentration : 1e-9);
  const double cold_mass = (h == E) ? 0.0 : (1.0 - (hot_mass < 1.0 ? hot_mass : 1.0));
  for (uint64_t it = 0; it < iters; ++it) {
    for (uint32_t l = 0; l < L; ++l) {
      uint32_t* hl = hot + (size_t)l * ORC_MAX_E;
      if (it > 0) evolve_hot(hl, h, E, persistence, &rng);
      double w[ORC_MAX_E], sum = 0.0;
      for (uint32_t i = 0; i < h; ++i) { w[i] = orc_rng_gamma(&rng, hot_shape); sum += w[i]; }
      for (uint32_t i = 0; i < h; ++i) w[i] = sum > 0.0 ? w[i] / sum * hot_mass : 0.0;
      for (uint32_t t = 0; t < B; ++t) {
        double* s = out + (((size_t)it * L + l) * B + t) * E;
        uint8_t is_hot[ORC_MAX_E];
        memset(is_hot, 0, E);
        for (uint32_t e = 0; e < E; ++e) s[e] = 0.0;
        for (uint32_t i = 0; i < h; ++i) { is_hot[hl[i]] = 1; s[hl[i]] = w[i]; }
        double cold[ORC_MAX_E], csum = 0.0;
        for (uint32_t e = 0; e < E; ++e) {
          cold[e] = 0.0;
          if (!is_hot[e]) { cold[e] = orc_rng_gamma(&rng, 2.0); csum += cold[e]; }
        }
        for (uint32_t e = 0; e < E; ++e)
          if (!is_hot[e]) s[e] = csum > 0.0 ? cold[e] / csum * cold_mass : 0.0;
      }
    }
  }
  free(hot);
}

/* ---------------------------------------------------------------- cache */
typedef struct orc_layer {
  uint32_t n_res;
  uint32_t res[ORC_MAX_E]; /* sorted ascending */
  uint8_t mask[ORC_MAX_E];
  uint8_t shield[ORC_MAX_E];
  uint64_t last[ORC_MAX_E];
  double* hist; /* ring [window][E] */
  uint32_t h_head, h_size; /* oldest at h_head */
} orc_layer;

struct orc_cache {
  uint32_t L, E, slots, window;
  int32_t policy;
  orc_layer* layers;
};

/* cache.cpp:10-44 */
orc_cache* orc_cache_new(uint32_t L, uint32_t E, uint32_t slots, uint32_t window, int32_t policy,
                         int32_t init_fill, uint64_t seed) {
  orc_cache* c = (orc_cache*)calloc(1, sizeof *c);
  c->L = L; c->E = E; c->slots = slots; c->window = window; c->policy = policy;
  c->layers = (orc_layer*)calloc(L, sizeof(orc_layer));
  const uint32_t cap = slots < E ? slots : E;
  for (uint32_t l = 0; l < L; ++l) {
    orc_layer* ly = &c->layers[l];
    ly->hist = (double*)calloc((size_t)window * E + 1, sizeof(double));
    if (init_fill == 1) {
      orc_rng rng;
      orc_rng_seed(&rng, orc_derive_seed(seed, 0x11caffe0ULL + l));
      uint32_t pool[ORC_MAX_E];
      for (uint32_t i = 0; i < E; ++i) pool[i] = i;
      for (uint32_t i = 0; i < cap; ++i) {
        const uint64_t j = i + orc_rng_below(&rng, E - i);
        const uint32_t tmp = pool[i];
        pool[i] = pool[j];
        pool[j] = tmp;
        ly->res[ly->n_res++] = pool[i];
      }
      sort_u32(ly->res, ly->n_res);
    } else if (init_fill == 0) {
      for (uint32_t i = 0; i < cap; ++i) ly->res[ly->n_res++] = i;
    }
    for (uint32_t i = 0; i < ly->n_res; ++i) ly->mask[ly->res[i]] = 1;
  }
  return c;
}
void orc_cache_free(orc_cache* c) {
  if (!c) return;
  for (uint32_t l = 0; l < c->L; ++l) free(c->layers[l].hist);
  free(c->layers);
  free(c);
}
uint32_t orc_cache_resident(const orc_cache* c, uint32_t layer, uint32_t* out) {
  const orc_layer* ly = &c->layers[layer];
  if (out) memcpy(out, ly->res, ly->n_res * sizeof(uint32_t));
  return ly->n_res;
}
/* cache.cpp:58-67 */
int orc_cache_record(orc_cache* c, uint32_t layer, const double* s, uint32_t n) {
  if (n != c->E) return ORC_ELOGIC;
  orc_layer* ly = &c->layers[layer];
  uint32_t slot;
  if (ly->h_size < c->window) {
    slot = (ly->h_head + ly->h_size) % c->window;
    ly->h_size++;
  } else {
    slot = ly->h_head; /* overwrite oldest = push_back + pop_front */
    ly->h_head = (ly->h_head + 1) % c->window;
  }
  memcpy(ly->hist + (size_t)slot * c->E, s, c->E * sizeof(double));
  return ORC_OK;
}
/* cache.cpp:69-79 — oldest to newest, then divide by size */
double orc_cache_window_average(const orc_cache* c, uint32_t layer, uint32_t e) {
  const orc_layer* ly = &c->layers[layer];
  if (ly->h_size == 0) return 0.0;
  double sum = 0.0;
  for (uint32_t i = 0; i < ly->h_size; ++i)
    sum += ly->hist[(size_t)((ly->h_head + i) % c->window) * c->E + e];
  return sum / (double)ly->h_size;
}
/* cache.cpp:81-109 */
int64_t orc_cache_try_evict(const orc_cache* c, uint32_t layer) {
  const orc_layer* ly = &c->layers[layer];
  int64_t victim = -1;
  if (c->policy == 0) {
    double best = 0.0;
    for (uint32_t i = 0; i < ly->n_res; ++i) {
      const uint32_t e = ly->res[i];
      if (ly->shield[e]) continue;
      const double a = orc_cache_window_average(c, layer, e);
      if (victim < 0 || a < best) { victim = e; best = a; }
    }
  } else {
    uint64_t best = 0;
    for (uint32_t i = 0; i < ly->n_res; ++i) {
      const uint32_t e = ly->res[i];
      if (ly->shield[e]) continue;
      if (victim < 0 || ly->last[e] < best) { victim = e; best = ly->last[e]; }
    }
  }
  return victim;
}
/* cache.cpp:119-134 */
void orc_cache_shield(orc_cache* c, uint32_t layer, uint32_t e) { c->layers[layer].shield[e] = 1; }
void orc_cache_unshield(orc_cache* c, uint32_t layer) {
  memset(c->layers[layer].shield, 0, sizeof c->layers[layer].shield);
}
int orc_cache_is_shielded(const orc_cache* c, uint32_t layer, uint32_t e) {
  return c->layers[layer].shield[e] != 0;
}
void orc_cache_touch(orc_cache* c, uint32_t layer, uint32_t e, uint64_t now) {
  c->layers[layer].last[e] = now;
}
/* cache.cpp:136-156 */
int orc_cache_admit(orc_cache* c, uint32_t layer, uint32_t e, uint64_t now, int64_t* evicted) {
  orc_layer* ly = &c->layers[layer];
  *evicted = -1;
  if (ly->mask[e]) return ORC_ELOGIC;
  if (c->slots == 0) return ORC_OK;
  if (ly->n_res >= c->slots) {
    const int64_t v = orc_cache_try_evict(c, layer);
    if (v < 0) return ORC_ECACHE;
    uint32_t w = 0;
    for (uint32_t i = 0; i < ly->n_res; ++i)
      if (ly->res[i] != (uint32_t)v) ly->res[w++] = ly->res[i];
    ly->n_res = w;
    ly->mask[v] = 0;
    *evicted = v;
  }
  uint32_t pos = ly->n_res;
  while (pos > 0 && ly->res[pos - 1] > e) { ly->res[pos] = ly->res[pos - 1]; --pos; }
  ly->res[pos] = e;
  ly->n_res++;
  ly->mask[e] = 1;
  ly->last[e] = now;
  return ORC_OK;
}

/* -------------------------------------------------------- JSON builder */
typedef struct jbuf { char* p; size_t n, cap; } jbuf;
static void jb_put(jbuf* b, const char* fmt, ...) {
  va_list ap;
  for (;;) {
    va_start(ap, fmt);
    const int w = vsnprintf(b->p + b->n, b->cap - b->n, fmt, ap);
    va_end(ap);
    if (w >= 0 && (size_t)w < b->cap - b->n) { b->n += (size_t)w; return; }
    b->cap = b->cap * 2 + (size_t)(w > 0 ? w : 64) + 64;
    b->p = (char*)realloc(b->p, b->cap);
  }
}
static void jb_list(jbuf* b, const uint32_t* v, uint32_t n) {
  jb_put(b, "[");
  for (uint32_t i = 0; i < n; ++i) jb_put(b, i ? ",%u" : "%u", v[i]);
  jb_put(b, "]");
}

/* ------------------------------------------------------------- pipeline */
enum { RES_GPU = 0, RES_CPU = 1, RES_PCIE = 2 };
enum { K_ATTN = 0, K_ROUTE, K_RESIDENT, K_LOADED, K_CPU, K_DEMAND, K_PREFETCH };

typedef struct orc_task {
  uint8_t res, kind;
  int32_t elayer; /* -1 = no expert */
  uint32_t eidx;
  uint64_t start, end;
  uint32_t layer;
  uint64_t it;
} orc_task;

typedef struct orc_sim {
  const orc_config* cfg;
  const double* scores;
  const double* pred;
  const uint8_t* has_pred;
  uint64_t iters;
  orc_cache* cache;
  orc_rng prng;
  uint64_t gpu_free, cpu_free, pcie_free;
  /* prefetch queue (pipeline.cpp:159) */
  int q_valid;
  uint32_t q_layer;
  uint64_t q_it;
  uint32_t q_n;
  uint32_t q_e[ORC_MAX_E];
  uint8_t q_issued[ORC_MAX_E];
  /* deferred admissions (pipeline.cpp:162) */
  uint32_t n_def;
  uint32_t def_l[ORC_MAX_E * 8], def_e[ORC_MAX_E * 8];
  /* metrics (pipeline.hpp:63-78) */
  uint64_t demand, prefetch, cpu_computed, hits, misses, subs, kept_low, selections;
  /* PredictorStats (prefetch.hpp:68-88) */
  uint64_t draws, trace_supplied, head_top, head_active, head_inactive, issued, cancelled;
  /* logs */
  int emit_tl, emit_steps;
  orc_task* tasks;
  size_t n_tasks, cap_tasks;
  jbuf win, ev, steps;
  int n_win, n_ev, n_steps;
  /* per-step record scratch */
  uint32_t st_pref[ORC_MAX_E], st_npref;
  uint32_t st_evict[ORC_MAX_E * 8][2], st_nevict;
} orc_sim;

static void push_task(orc_sim* S, int res, int kind, int32_t el, uint32_t ei, uint64_t s,
                      uint64_t e, uint32_t layer, uint64_t it) {
  if (!S->emit_tl) return;
  if (S->n_tasks == S->cap_tasks) {
    S->cap_tasks = S->cap_tasks ? S->cap_tasks * 2 : 4096;
    S->tasks = (orc_task*)realloc(S->tasks, S->cap_tasks * sizeof(orc_task));
  }
  orc_task* t = &S->tasks[S->n_tasks++];
  t->res = (uint8_t)res; t->kind = (uint8_t)kind; t->elayer = el; t->eidx = ei;
  t->start = s; t->end = e; t->layer = layer; t->it = it;
}

static const double* sc_at(const orc_sim* S, uint64_t it, uint32_t layer) {
  const orc_config* c = S->cfg;
  return S->scores + (((size_t)it * c->num_layers + layer) * c->batch) * c->experts;
}

/* pipeline.cpp:93-108 */
static void admit_or_defer(orc_sim* S, uint32_t layer, uint32_t e, uint64_t now, int shield) {
  orc_layer* ly = &S->cache->layers[layer];
  if (ly->mask[e]) return;
  int64_t ev;
  const int rc = orc_cache_admit(S->cache, layer, e, now, &ev);
  if (rc == ORC_ECACHE) {
    S->def_l[S->n_def] = layer;
    S->def_e[S->n_def] = e;
    S->n_def++;
    return;
  }
  if (ev >= 0) {
    if (S->emit_tl) {
      jb_put(&S->ev, "%s[%llu,%u,%lld]", S->n_ev ? "," : "", (unsigned long long)now, layer,
             (long long)ev);
      S->n_ev++;
    }
    if (S->st_nevict < ORC_MAX_E * 8) {
      S->st_evict[S->st_nevict][0] = layer;
      S->st_evict[S->st_nevict][1] = (uint32_t)ev;
      S->st_nevict++;
    }
  }
  if (shield) orc_cache_shield(S->cache, layer, e);
}

/* pipeline.cpp:293-344 */
static int schedule_prefetch(orc_sim* S, uint64_t it, uint32_t layer, uint64_t resident_done,
                             uint64_t completion) {
  const orc_config* c = S->cfg;
  uint64_t tit = it;
  uint32_t tl = layer + 1;
  if (tl == c->num_layers) { tl = 0; ++tit; }
  if (tit >= S->iters) return ORC_OK;
  const uint64_t gate = completion + c->t_attn;
  const uint32_t E = c->experts;
  double merged[ORC_MAX_E];
  for (uint32_t e = 0; e < E; ++e) merged[e] = 0.0;
  const double* ts = sc_at(S, tit, tl);
  for (uint32_t t = 0; t < c->batch; ++t) {
    const size_t row = ((size_t)tit * c->num_layers + tl) * c->batch + t;
    const double* sup = (S->pred && S->has_pred && S->has_pred[row]) ? S->pred + row * E : NULL;
    double out[ORC_MAX_E];
    uint32_t head;
    int32_t kind;
    const int rc = orc_predict_scores(ts + (size_t)t * E, sup, E, c->p_top, c->p_active, c->top_k,
                                      c->alpha, &S->prng, out, &head, &kind);
    if (rc) return rc;
    if (sup) S->trace_supplied++; else S->draws++;
    if (kind == 0) S->head_top++; else if (kind == 1) S->head_active++; else S->head_inactive++;
    for (uint32_t e = 0; e < E; ++e) merged[e] = merged[e] > out[e] ? merged[e] : out[e];
  }
  const uint32_t depth = c->queue_depth == 0 ? c->top_k : c->queue_depth;
  orc_layer* ly = &S->cache->layers[tl];
  uint32_t ent[ORC_MAX_E], ne;
  orc_build_queue(merged, ly->mask, E, depth, ent, &ne);
  S->q_valid = 1; S->q_layer = tl; S->q_it = tit; S->q_n = ne;
  uint64_t t = S->pcie_free > resident_done ? S->pcie_free : resident_done;
  for (uint32_t i = 0; i < ne; ++i) {
    S->q_e[i] = ent[i];
    S->q_issued[i] = 0;
  }
  for (uint32_t i = 0; i < ne; ++i) {
    if (t + c->t_load > gate) break;
    if (ly->mask[ent[i]]) continue;
    push_task(S, RES_PCIE, K_PREFETCH, (int32_t)tl, ent[i], t, t + c->t_load, tl, tit);
    t += c->t_load;
    S->q_issued[i] = 1;
    S->issued++;
    S->prefetch++;
    S->st_pref[S->st_npref++] = ent[i];
    admit_or_defer(S, tl, ent[i], t, 0);
  }
  if (t > S->pcie_free) S->pcie_free = t;
  return ORC_OK;
}

/* pipeline.cpp:128-286 */
static int run_layer(orc_sim* S, uint64_t it, uint32_t layer, uint64_t start, uint64_t* done) {
  const orc_config* c = S->cfg;
  const uint32_t E = c->experts, B = c->batch, k = c->top_k;
  const double* bs = sc_at(S, it, layer);
  orc_layer* ly = &S->cache->layers[layer];
  S->st_npref = 0;
  S->st_nevict = 0;

  const uint64_t attn_end = start + c->t_attn;
  push_task(S, RES_GPU, K_ATTN, -1, 0, start, attn_end, layer, it);
  S->gpu_free = attn_end;
  if (S->q_valid && S->q_layer == layer && S->q_it == it) {
    for (uint32_t i = 0; i < S->q_n; ++i) S->cancelled += !S->q_issued[i];
    S->q_valid = 0;
  }
  const uint64_t route_start = attn_end > S->cpu_free ? attn_end : S->cpu_free;
  const uint64_t route_end = route_start + c->t_route;
  push_task(S, RES_CPU, K_ROUTE, -1, 0, route_start, route_end, layer, it);
  S->cpu_free = route_end;

  uint8_t mask[ORC_MAX_E];
  memcpy(mask, ly->mask, E);

  orc_token_route* toks = (orc_token_route*)malloc(sizeof(orc_token_route) * (B ? B : 1));
  if (c->er) {
    uint32_t cset[ORC_MAX_E], nc, pend[ORC_MAX_E], np;
    int rc = orc_route(bs, B, E, mask, k, c->alpha, toks, cset, &nc, pend, &np);
    if (rc) { free(toks); return rc; }
    orc_coalesce(toks, bs, B, E, mask, cset, nc, pend, &np);
    for (uint32_t t = 0; t < B; ++t) { S->subs += toks[t].n_sub; S->kept_low += toks[t].n_kept; }
  } else {
    for (uint32_t t = 0; t < B; ++t) {
      orc_plain_top_k(bs + (size_t)t * E, E, k, toks[t].sel, &toks[t].n_sel);
      toks[t].n_sub = toks[t].n_kept = 0;
    }
  }
  uint32_t cnt[ORC_MAX_E];
  memset(cnt, 0, sizeof cnt);
  for (uint32_t t = 0; t < B; ++t)
    for (uint32_t i = 0; i < toks[t].n_sel; ++i) {
      const uint32_t e = toks[t].sel[i];
      S->selections++;
      if (mask[e]) S->hits++; else S->misses++;
      cnt[e]++;
    }
  /* pipeline.cpp:79-91 mean over tokens, token order, then / B */
  double mean[ORC_MAX_E];
  for (uint32_t e = 0; e < E; ++e) mean[e] = 0.0;
  for (uint32_t t = 0; t < B; ++t)
    for (uint32_t e = 0; e < E; ++e) mean[e] += bs[(size_t)t * E + e];
  for (uint32_t e = 0; e < E; ++e) mean[e] /= (double)B;
  orc_cache_record(S->cache, layer, mean, E);

  uint32_t distinct[ORC_MAX_E], nd = 0, resd[ORC_MAX_E], nr = 0;
  uint32_t duid[ORC_MAX_E], dbat[ORC_MAX_E], ndm = 0;
  for (uint32_t e = 0; e < E; ++e) {
    if (!cnt[e]) continue;
    distinct[nd++] = e;
    if (mask[e]) {
      resd[nr++] = e;
      orc_cache_shield(S->cache, layer, e);
      orc_cache_touch(S->cache, layer, e, route_end);
    } else {
      duid[ndm] = e;
      dbat[ndm] = cnt[e];
      ndm++;
    }
  }
  uint32_t load[ORC_MAX_E], nl = 0, cpu[ORC_MAX_E], ncpu = 0;
  if (c->ba) {
    uint64_t cl, cc;
    orc_balance(duid, dbat, ndm, c->t_cpu_token, c->t_load, load, &nl, cpu, &ncpu, &cl, &cc);
  } else {
    for (uint32_t i = 0; i < ndm; ++i) load[nl++] = duid[i];
  }
  uint64_t cpu_t = route_end > S->cpu_free ? route_end : S->cpu_free;
  for (uint32_t i = 0; i < ncpu; ++i) {
    const uint64_t dur = (uint64_t)cnt[cpu[i]] * c->t_cpu_token;
    push_task(S, RES_CPU, K_CPU, (int32_t)layer, cpu[i], cpu_t, cpu_t + dur, layer, it);
    cpu_t += dur;
    S->cpu_computed++;
  }
  S->cpu_free = cpu_t;

  uint64_t ready[ORC_MAX_E];
  uint64_t pcie_t = route_end > S->pcie_free ? route_end : S->pcie_free;
  for (uint32_t i = 0; i < nl; ++i) {
    push_task(S, RES_PCIE, K_DEMAND, (int32_t)layer, load[i], pcie_t, pcie_t + c->t_load, layer, it);
    pcie_t += c->t_load;
    admit_or_defer(S, layer, load[i], pcie_t, 1);
    ready[i] = pcie_t;
    S->demand++;
  }
  S->pcie_free = pcie_t;

  uint64_t gpu_t = S->gpu_free > route_end ? S->gpu_free : route_end;
  uint64_t resident_done = attn_end > route_end ? attn_end : route_end;
  for (uint32_t i = 0; i < nr; ++i) {
    push_task(S, RES_GPU, K_RESIDENT, (int32_t)layer, resd[i], gpu_t, gpu_t + c->t_gpu, layer, it);
    gpu_t += c->t_gpu;
  }
  if (nr) resident_done = gpu_t;
  for (uint32_t i = 0; i < nl; ++i) {
    const uint64_t s0 = gpu_t > ready[i] ? gpu_t : ready[i];
    push_task(S, RES_GPU, K_LOADED, (int32_t)layer, load[i], s0, s0 + c->t_gpu, layer, it);
    gpu_t = s0 + c->t_gpu;
  }
  S->gpu_free = gpu_t;
  uint64_t completion = attn_end;
  if (route_end > completion) completion = route_end;
  if (S->cpu_free > completion) completion = S->cpu_free;
  if ((nr || nl) && gpu_t > completion) completion = gpu_t;

  if (S->emit_tl) {
    jb_put(&S->win, "%s[%llu,%u,%llu,%llu,%llu,", S->n_win ? "," : "", (unsigned long long)it,
           layer, (unsigned long long)attn_end, (unsigned long long)route_end,
           (unsigned long long)completion);
    jb_list(&S->win, distinct, nd);
    jb_put(&S->win, "]");
    S->n_win++;
  }

  orc_cache_unshield(S->cache, layer);
  const uint32_t nd0 = S->n_def;
  uint32_t dl[ORC_MAX_E * 8], de[ORC_MAX_E * 8];
  memcpy(dl, S->def_l, nd0 * sizeof(uint32_t));
  memcpy(de, S->def_e, nd0 * sizeof(uint32_t));
  S->n_def = 0;
  for (uint32_t i = 0; i < nd0; ++i) admit_or_defer(S, dl[i], de[i], completion, 0);

  if (c->pre) {
    const int rc = schedule_prefetch(S, it, layer, resident_done, completion);
    if (rc) { free(toks); return rc; }
  }

  if (S->emit_steps) {
    jb_put(&S->steps, "%s{\"it\":%llu,\"layer\":%u,\"mask\":", S->n_steps ? "," : "",
           (unsigned long long)it, layer);
    uint32_t ml[ORC_MAX_E], nm = 0;
    for (uint32_t e = 0; e < E; ++e)
      if (mask[e]) ml[nm++] = e;
    jb_list(&S->steps, ml, nm);
    jb_put(&S->steps, ",\"tok\":[");
    for (uint32_t t = 0; t < B; ++t) {
      jb_put(&S->steps, "%s{\"sel\":", t ? "," : "");
      jb_list(&S->steps, toks[t].sel, toks[t].n_sel);
      jb_put(&S->steps, ",\"sub\":[");
      for (uint32_t i = 0; i < toks[t].n_sub; ++i)
        jb_put(&S->steps, "%s[%u,%u]", i ? "," : "", toks[t].sub_dropped[i], toks[t].sub_chosen[i]);
      jb_put(&S->steps, "],\"kept\":");
      jb_list(&S->steps, toks[t].kept, toks[t].n_kept);
      jb_put(&S->steps, "}");
    }
    jb_put(&S->steps, "],\"load\":");
    jb_list(&S->steps, load, nl);
    jb_put(&S->steps, ",\"cpu\":");
    jb_list(&S->steps, cpu, ncpu);
    jb_put(&S->steps, ",\"pref\":");
    jb_list(&S->steps, S->st_pref, S->st_npref);
    jb_put(&S->steps, ",\"evict\":[");
    for (uint32_t i = 0; i < S->st_nevict; ++i)
      jb_put(&S->steps, "%s[%u,%u]", i ? "," : "", S->st_evict[i][0], S->st_evict[i][1]);
    jb_put(&S->steps, "],\"completion\":%llu}", (unsigned long long)completion);
    S->n_steps++;
  }
  free(toks);
  *done = completion;
  return ORC_OK;
}

static int task_cmp(const void* a, const void* b) {
  const orc_task* x = (const orc_task*)a;
  const orc_task* y = (const orc_task*)b;
#define CMP(f) if (x->f != y->f) return x->f < y->f ? -1 : 1;
  CMP(start) CMP(res) CMP(end) CMP(layer) CMP(it) CMP(kind) CMP(elayer) CMP(eidx)
#undef CMP
  return 0;
}

static const char* kVio = NULL;
/* core.cpp:30-70 (violations only; warnings are not decisions) */
static const char* first_violation(const orc_config* c) {
  if (c->num_layers == 0) return "shape.num_layers: must be >= 1";
  if (c->experts == 0) return "shape.experts_per_layer: must be >= 1";
  if (c->top_k == 0) return "shape.top_k: must be >= 1";
  if (c->batch == 0) return "shape.batch_size: must be >= 1";
  if (c->top_k + 1 > c->experts) return "shape.top_k: k + 1 <= E required";
  if (!(c->alpha >= 0.0 && c->alpha < 1.0)) return "router.alpha: must satisfy 0 <= alpha < 1";
  if (c->slots > c->experts) return "cache.slots_per_layer: slots_per_layer <= E";
  if (c->window == 0) return "cache.history_window: must be >= 1";
  if (!(c->p_top >= 0.0 && c->p_top <= 1.0)) return "predictor.p_top: must be in [0, 1]";
  if (!(c->p_active >= 0.0 && c->p_active <= 1.0)) return "predictor.p_active: must be in [0, 1]";
  return kVio;
}

/* pipeline.cpp:110-126, 346-385 */
char* orc_simulate_json(const orc_config* cfg, const double* scores, const double* pred,
                        const uint8_t* has_pred, uint64_t iters, int32_t emit_steps,
                        int32_t emit_timeline) {
  jbuf out = {0};
  out.cap = 256;
  out.p = (char*)malloc(out.cap);
  out.p[0] = 0;
  const char* vio = first_violation(cfg);
  if (vio) { jb_put(&out, "{\"error\":\"invalid config: %s\"}", vio); return out.p; }
  if (cfg->experts > ORC_MAX_E) { jb_put(&out, "{\"error\":\"oracle: E too large\"}"); return out.p; }

  orc_sim S;
  memset(&S, 0, sizeof S);
  S.cfg = cfg; S.scores = scores; S.pred = pred; S.has_pred = has_pred; S.iters = iters;
  S.emit_tl = emit_timeline; S.emit_steps = emit_steps;
  /* pipeline.cpp:64-70: CE off => LRU */
  const int32_t policy = cfg->ce ? cfg->policy : 1;
  S.cache = orc_cache_new(cfg->num_layers, cfg->experts, cfg->slots, cfg->window, policy,
                          cfg->init_fill, cfg->seed);
  orc_rng_seed(&S.prng, orc_derive_seed(cfg->seed, 0x94ed1c70ULL));
  S.win.cap = S.ev.cap = S.steps.cap = 1024;
  S.win.p = (char*)calloc(1, 1024); S.ev.p = (char*)calloc(1, 1024); S.steps.p = (char*)calloc(1, 1024);

  uint64_t now = 0;
  jbuf itc = {0};
  itc.cap = 1024; itc.p = (char*)calloc(1, 1024);
  int rc = ORC_OK;
  for (uint64_t it = 0; it < iters && rc == ORC_OK; ++it) {
    for (uint32_t l = 0; l < cfg->num_layers && rc == ORC_OK; ++l) rc = run_layer(&S, it, l, now, &now);
    if (emit_timeline) jb_put(&itc, "%s%llu", it ? "," : "", (unsigned long long)now);
  }
  if (rc != ORC_OK) {
    jb_put(&out, "{\"error\":\"classify: beta undefined, need at least k+1 experts\"}");
  } else {
    const double tpot = iters ? (double)now / (double)iters : 0.0;
    const double hr = S.selections ? (double)S.hits / (double)S.selections : 0.0;
    const uint64_t st = S.subs + S.kept_low;
    const double sr = st ? (double)S.subs / (double)st : 0.0;
    jb_put(&out,
           "{\"metrics\":{\"tpot\":%.17g,\"hit_rate\":%.17g,\"substitution_ratio\":%.17g,"
           "\"demand_loads\":%llu,\"prefetch_loads\":%llu,\"cpu_computed\":%llu,\"hits\":%llu,"
           "\"misses\":%llu,\"substitutions\":%llu,\"low_score_kept\":%llu,\"selections\":%llu,"
           "\"iterations\":%llu,\"total_time\":%llu},",
           tpot, hr, sr, (unsigned long long)S.demand, (unsigned long long)S.prefetch,
           (unsigned long long)S.cpu_computed, (unsigned long long)S.hits,
           (unsigned long long)S.misses, (unsigned long long)S.subs,
           (unsigned long long)S.kept_low, (unsigned long long)S.selections,
           (unsigned long long)iters, (unsigned long long)now);
    jb_put(&out,
           "\"stats\":{\"draws\":%llu,\"trace_supplied\":%llu,\"head_top\":%llu,"
           "\"head_active\":%llu,\"head_inactive\":%llu,\"issued\":%llu,\"cancelled\":%llu},",
           (unsigned long long)S.draws, (unsigned long long)S.trace_supplied,
           (unsigned long long)S.head_top, (unsigned long long)S.head_active,
           (unsigned long long)S.head_inactive, (unsigned long long)S.issued,
           (unsigned long long)S.cancelled);
    jb_put(&out, "\"cache_final\":[");
    for (uint32_t l = 0; l < cfg->num_layers; ++l) {
      if (l) jb_put(&out, ",");
      jb_list(&out, S.cache->layers[l].res, S.cache->layers[l].n_res);
    }
    jb_put(&out, "]");
    if (emit_timeline) {
      qsort(S.tasks, S.n_tasks, sizeof(orc_task), task_cmp);
      jb_put(&out, ",\"tasks\":[");
      for (size_t i = 0; i < S.n_tasks; ++i) {
        const orc_task* t = &S.tasks[i];
        jb_put(&out, "%s[%u,%u,%d,%u,%llu,%llu,%u,%llu]", i ? "," : "", t->res, t->kind,
               t->elayer, t->eidx, (unsigned long long)t->start, (unsigned long long)t->end,
               t->layer, (unsigned long long)t->it);
      }
      jb_put(&out, "],\"windows\":[%s],\"evictions\":[%s],\"iteration_completion\":[%s]",
             S.win.p, S.ev.p, itc.p);
    }
    if (emit_steps) jb_put(&out, ",\"steps\":[%s]", S.steps.p);
    jb_put(&out, "}");
  }
  free(S.tasks);
  free(S.win.p); free(S.ev.p); free(S.steps.p); free(itc.p);
  orc_cache_free(S.cache);
  return out.p;
}

void orc_free(void* p) { free(p); }
