// C entry points over the REFERENCE's own RNG (proj/src/core/rng.cpp),
// compiled from /root/reference where it lies into oracle/_ref/ (never copied).
// Test infrastructure only: used to pin the oracle's and the device's
// xoshiro256** / split / uniform streams bit-for-bit (tests/golden/).
#include "core/rng.hpp"

#include <cstdint>

extern "C" {

// Draws `n` values from Rng(seed).split(k0,k1,k2) (or Rng(seed) when
// split==0): kind 0 = next_u64, 1 = uniform() bits, 2 = uniform_int(m), 3 = normal() bits.
void ref_rng_draw(std::uint64_t seed, int split, std::uint64_t k0, std::uint64_t k1,
                  std::uint64_t k2, int kind, std::uint64_t m, std::uint64_t* out,
                  std::size_t n) {
  b3d::Rng base(seed);
  b3d::Rng r = split ? base.split(k0, k1, k2) : base;
  for (std::size_t i = 0; i < n; ++i) {
    if (kind == 0) {
      out[i] = r.next_u64();
    } else if (kind == 1) {
      double u = r.uniform();
      __builtin_memcpy(&out[i], &u, 8);
    } else if (kind == 2) {
      out[i] = r.uniform_int(m);
    } else {
      double g = r.normal();
      __builtin_memcpy(&out[i], &g, 8);
    }
  }
}
}
