// Frozen SplitMix64 stream, tag mixing and Box-Muller Gaussian blocks.
//
// Follows proj/include/hpeel/rng.hpp:12-48 and proj/src/rng.cpp:8-59. The
// stream is counter-addressable (after n draws the state is seed + n*gamma),
// so entry (i, j) of a rows x cols Gaussian block is a pure function of
// (seed, i*cols + j); `gaussian_entry` is shared by the host and the device
// payload kernel (K1) so both read the same stream positions.
#pragma once

#include <cmath>
#include <cstdint>

#include "matrix.hpp"

#ifdef __CUDACC__
#define HP_HD __host__ __device__ __forceinline__
#else
#define HP_HD inline
#endif

namespace hpeel {

constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ull;

HP_HD std::uint64_t scramble(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : state_(seed) {}
  std::uint64_t next() {
    state_ += kGamma;
    return scramble(state_);
  }
  double next_open_closed() { return double((next() >> 11) + 1) * 0x1.0p-53; }
  double next_closed_open() { return double(next() >> 11) * 0x1.0p-53; }

 private:
  std::uint64_t state_;
};

HP_HD std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t tag) {
  return scramble(seed * kGamma + tag + 1);
}
HP_HD std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t t1, std::uint64_t t2) {
  return mix_seed(mix_seed(seed, t1), t2);
}
HP_HD std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t t1, std::uint64_t t2,
                             std::uint64_t t3) {
  return mix_seed(mix_seed(mix_seed(seed, t1), t2), t3);
}

/// Element e = i*cols + j of the row-major Box-Muller stream with the given
/// seed (proj/src/rng.cpp:42-57): pair q = e/2 draws u1 = next_open_closed at
/// stream position 2q+1 and u2 = next_closed_open at 2q+2; even e takes the
/// cosine variate, odd e the sine variate.
HP_HD double gaussian_entry(std::uint64_t seed, std::uint64_t e) {
  const std::uint64_t q = e >> 1;
  const std::uint64_t s1 = scramble(seed + (2 * q + 1) * kGamma);
  const std::uint64_t s2 = scramble(seed + (2 * q + 2) * kGamma);
  const double u1 = double((s1 >> 11) + 1) * 0x1.0p-53;
  const double u2 = double(s2 >> 11) * 0x1.0p-53;
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * M_PI * u2;
  return (e & 1) ? radius * sin(angle) : radius * cos(angle);
}

/// rows x cols standard-normal matrix, row-major stream order
/// (proj/src/rng.cpp:35-59).
Matrix gaussian_matrix(Index rows, Index cols, std::uint64_t seed);

/// Payload seed of box `box` at (level, phase): proj/src/coloring.cpp:252-259.
HP_HD std::uint64_t payload_seed(std::uint64_t seed, int level, int box, int phase) {
  return mix_seed(seed, std::uint64_t(level), std::uint64_t(box), std::uint64_t(phase));
}

}  // namespace hpeel
