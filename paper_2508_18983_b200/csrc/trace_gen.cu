// trace_gen.cu — synthetic gate-score streams (GateTrace workload generator).
//
// Host-side restatement of generate_trace (trace.cpp:106-151): per layer a
// Markov-persistent hot set, per (iteration, layer) hot weights shared by the
// batch's tokens, per token a cold Dirichlet tier. This is workload
// synthesis (it produces the router logits the bench and the stack consume),
// not part of the device hot path; it reuses the engine's bit-exact RNG.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/moesched_b200.h"
#include "engine.cuh"
#include "host_common.h"

namespace moeb {
namespace {

struct HostRng {
  uint64_t s[4];
  explicit HostRng(uint64_t seed) { rng_seed(s, seed); }
  uint64_t u64() { return rng_u64(s); }
  double uniform() { return rng_double(s); }
  uint64_t below(uint64_t n) { return rng_below(s, n); }
  // rng.cpp:58-64 Box-Muller, second variate discarded
  double normal() {
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
  }
  // rng.cpp:66-89 Marsaglia-Tsang with the shape<1 boost
  double gamma(double shape) {
    if (shape < 1.0) {
      const double u = 1.0 - uniform();
      return gamma(shape + 1.0) * std::pow(u, 1.0 / shape);
    }
    const double d = shape - 1.0 / 3.0;
    const double c = 1.0 / std::sqrt(9.0 * d);
    for (;;) {
      const double x = normal();
      const double t = 1.0 + c * x;
      if (t <= 0.0) continue;
      const double v = t * t * t;
      const double u = uniform();
      if (u < 1.0 - 0.0331 * x * x * x * x) return d * v;
      if (u > 0.0 && std::log(u) < 0.5 * x * x + d * (1.0 - v + std::log(v))) return d * v;
    }
  }
};

}  // namespace

void generate_trace_host(uint32_t L, uint32_t E, uint32_t B, double hot_fraction, double hot_mass,
                         double persistence, double concentration, uint64_t iters, uint64_t seed,
                         double* out) {
  HostRng rng(derive_seed(seed, 0x7ace5eedULL));
  const long hl = std::lround(hot_fraction * (double)E);
  const uint32_t h = std::clamp<uint32_t>(static_cast<uint32_t>(hl), 1u, E);
  std::vector<std::vector<uint32_t>> hot(L);
  for (uint32_t l = 0; l < L; ++l) {
    std::vector<uint32_t> pool(E);
    for (uint32_t i = 0; i < E; ++i) pool[i] = i;
    for (uint32_t i = 0; i < h; ++i) {
      const uint64_t j = i + rng.below(E - i);
      std::swap(pool[i], pool[j]);
      hot[l].push_back(pool[i]);
    }
    std::sort(hot[l].begin(), hot[l].end());
  }
  const double hot_shape = 1.0 / std::max(concentration, 1e-9);
  const double cold_mass = (h == E) ? 0.0 : (1.0 - std::min(hot_mass, 1.0));
  std::vector<uint8_t> in_new(E), is_hot(E);
  std::vector<double> cold(E), w(E);
  for (uint64_t it = 0; it < iters; ++it) {
    for (uint32_t l = 0; l < L; ++l) {
      std::vector<uint32_t>& hs = hot[l];
      if (it > 0) {
        // trace.cpp:26-51: keep with prob persistence, refill uniformly
        std::fill(in_new.begin(), in_new.end(), 0);
        std::vector<uint32_t> kept;
        for (uint32_t e : hs)
          if (rng.uniform() < persistence) { kept.push_back(e); in_new[e] = 1; }
        const size_t need = hs.size() - kept.size();
        for (size_t i = 0; i < need; ++i) {
          std::vector<uint32_t> cand;
          for (uint32_t e = 0; e < E; ++e)
            if (!in_new[e]) cand.push_back(e);
          const uint32_t pick = cand[rng.below(cand.size())];
          kept.push_back(pick);
          in_new[pick] = 1;
        }
        std::sort(kept.begin(), kept.end());
        hs = kept;
      }
      double sum = 0.0;
      for (size_t i = 0; i < hs.size(); ++i) { w[i] = rng.gamma(hot_shape); sum += w[i]; }
      for (size_t i = 0; i < hs.size(); ++i) w[i] = sum > 0.0 ? w[i] / sum * hot_mass : 0.0;
      for (uint32_t t = 0; t < B; ++t) {
        double* s = out + (((size_t)it * L + l) * B + t) * E;
        std::fill(is_hot.begin(), is_hot.end(), 0);
        for (uint32_t e = 0; e < E; ++e) s[e] = 0.0;
        for (size_t i = 0; i < hs.size(); ++i) { is_hot[hs[i]] = 1; s[hs[i]] = w[i]; }
        double csum = 0.0;
        for (uint32_t e = 0; e < E; ++e) {
          cold[e] = 0.0;
          if (!is_hot[e]) { cold[e] = rng.gamma(2.0); csum += cold[e]; }
        }
        for (uint32_t e = 0; e < E; ++e)
          if (!is_hot[e]) s[e] = csum > 0.0 ? cold[e] / csum * cold_mass : 0.0;
      }
    }
  }
}

}  // namespace moeb

extern "C" int moeb_generate_trace(uint32_t L, uint32_t E, uint32_t B, double hot_fraction,
                                   double hot_mass, double persistence, double concentration,
                                   uint64_t iters, uint64_t seed, double* out) {
  return moeb::guarded([&] {
    if (E == 0 || L == 0 || B == 0) throw moeb::Error(1, "generate_trace: dimensions must be positive");
    moeb::generate_trace_host(L, E, B, hot_fraction, hot_mass, persistence, concentration, iters, seed, out);
  });
}
