// Host-side seeded initial-condition generator: xoshiro256++ seeded through
// splitmix64 with Box-Muller normals, bit-for-bit the reference's
// Xoshiro256pp / Uniform / Normal (models.py:43-130).  The reference runs this
// as a pure-Python loop (0.1 s per config-5 member); here it is plain C so a
// 512-member ensemble is generated in about a second.  Compiled with
// -ffp-contract=off so lo + (hi - lo) * u rounds exactly like NumPy.
#include <cmath>
#include <cstdint>

#include "curvigpu.h"

namespace {

inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

inline uint64_t next(uint64_t s[4]) {
  const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

constexpr double kTwoPow53Inv = 1.0 / 9007199254740992.0;  // 2^-53, exact

}  // namespace

extern "C" {

void cg_rng_seed(uint64_t seed, uint64_t state[4]) {
  uint64_t x = seed;
  for (int i = 0; i < 4; ++i) {
    x += 0x9E3779B97F4A7C15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    state[i] = z ^ (z >> 31);
  }
}

void cg_rng_next(uint64_t state[4], long long n, uint64_t* out) {
  for (long long i = 0; i < n; ++i) out[i] = next(state);
}

void cg_rng_uniform(uint64_t state[4], long long n, double lo, double hi, double* out) {
  const double span = hi - lo;
  for (long long i = 0; i < n; ++i) {
    const double u = static_cast<double>(next(state) >> 11) * kTwoPow53Inv;
    const double scaled = span * u;
    out[i] = lo + scaled;
  }
}

void cg_rng_normal(uint64_t state[4], long long n, double sigma, double* out) {
  const double two_pi = 2.0 * M_PI;
  long long i = 0;
  while (i < n) {
    const double u1 = static_cast<double>((next(state) >> 11) + 1) * kTwoPow53Inv;
    const double u2 = static_cast<double>(next(state) >> 11) * kTwoPow53Inv;
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double ang = two_pi * u2;
    out[i++] = sigma * (radius * std::cos(ang));
    if (i < n) out[i++] = sigma * (radius * std::sin(ang));
  }
}

}  // extern "C"
