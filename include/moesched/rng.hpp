// moesched/rng.hpp — drop-in re-declaration of the reference RNG
// (/root/reference/proj/include/moesched/rng.hpp:12-35): xoshiro256** seeded by
// splitmix64, bit-identical to the device engine's predictor stream.
#pragma once

#include <cstdint>

namespace moesched {

class Rng {
  public:
    explicit Rng(std::uint64_t seed);
    std::uint64_t next_u64();
    double next_double();                      // [0, 1), 53-bit
    std::uint64_t next_below(std::uint64_t n);  // unbiased, n > 0
    double next_normal();                      // Box-Muller, second variate dropped
    double next_gamma(double shape);           // Marsaglia-Tsang

    // B200 build: the xoshiro state, so device calls (predict_scores) can
    // advance the same stream.
    std::uint64_t* raw_state() { return state_; }

  private:
    std::uint64_t state_[4];
};

std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag);

}  // namespace moesched
