// Counter-based randomness shared by host and device code.
//
// Restates the published SplitMix64 finaliser and the reference's
// counter-keyed Gaussian stream (reference proj/core/include/etdec/rng.hpp:
// splitmix64 :15-20, mix_key :23-25, uniform_open01 :28-30, SplitMixEngine
// :34-65, NoiseStream :85-99) so that frame f's draws depend only on
// (seed, f, i): sharding frames over slots or GPUs never changes a draw.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define BPDEC_HD __host__ __device__ __forceinline__
#else
#define BPDEC_HD inline
#endif

namespace bpdec {

constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
// Key domain of NoiseStream (rng.hpp:87).
constexpr std::uint64_t kNoiseDomain = 0x243f6a8885a308d3ULL;
// Key domain of the message-bit stream x (new; BASELINE syndrome mode).
constexpr std::uint64_t kBitDomain = 0x13198a2e03707344ULL;
// Key domain of the per-frame efficiency draw (BASELINE config 5).
constexpr std::uint64_t kBetaDomain = 0xa4093822299f31d0ULL;

BPDEC_HD std::uint64_t splitmix64(std::uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

BPDEC_HD std::uint64_t mix_key(std::uint64_t key, std::uint64_t word) {
  return splitmix64(key ^ splitmix64(word));
}

// (0,1) open; 53-bit mantissa, never 0 or 1.
BPDEC_HD double uniform_open01(std::uint64_t word) {
  return (static_cast<double>(word >> 11) + 0.5) * 0x1.0p-53;
}

BPDEC_HD std::uint64_t stream_key(std::uint64_t domain, std::uint64_t seed, std::uint64_t stream) {
  return mix_key(mix_key(domain, seed), stream);
}

// Sequential generator for one-off seeded choices (code construction).
class SplitMixEngine {
 public:
  explicit SplitMixEngine(std::uint64_t seed) : state_(seed) {}
  std::uint64_t next() {
    state_ += kGolden;
    std::uint64_t z = state_;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  // Unbiased uniform in [0, n) by rejection over the next power-of-two mask.
  std::uint64_t bounded(std::uint64_t n) {
    std::uint64_t mask = n - 1;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    for (;;) {
      const std::uint64_t v = next() & mask;
      if (v < n) return v;
    }
  }

 private:
  std::uint64_t state_;
};

// The two uniforms of Box-Muller sample i of a stream keyed `key`
// (counters 2i and 2i+1).
BPDEC_HD void noise_uniforms(std::uint64_t key, std::uint64_t i, double* u1, double* u2) {
  *u1 = uniform_open01(splitmix64(key ^ splitmix64(2 * i)));
  *u2 = uniform_open01(splitmix64(key ^ splitmix64(2 * i + 1)));
}

// Per-frame reconciliation efficiency beta_f ~ U[lo, hi] keyed by (seed, f).
BPDEC_HD double frame_beta(std::uint64_t seed, std::uint64_t frame, double lo, double hi) {
  if (!(hi > lo)) return lo;
  const double u = uniform_open01(mix_key(mix_key(kBetaDomain, seed), frame));
  return lo + (hi - lo) * u;
}

// Message bit i of a stream keyed `key` (top bit of the hashed counter).
BPDEC_HD unsigned message_bit(std::uint64_t key, std::uint64_t i) {
  return static_cast<unsigned>(splitmix64(key ^ splitmix64(i)) >> 63);
}

}  // namespace bpdec
