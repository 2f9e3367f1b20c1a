// vmfa_rng.hpp — counter-based hashing and the xoshiro256++ stream used by the
// reference (rng.hpp:9-98), restated for host and device. The per-point extra
// candidate r_n = floor(hash3(seed, iteration, n) * C / 2^64) (rng.hpp:91-98)
// is evaluated on the device with __umul64hi, bit-identical to the reference's
// 128-bit multiply-high (pinned by tests/golden/rng_ref.json).
#pragma once
#include <cmath>
#include <cstdint>

#if defined(__CUDACC__)
#define VMFA_HD __host__ __device__ __forceinline__
#else
#define VMFA_HD inline
#endif

namespace vmfa_b200 {

VMFA_HD uint64_t sm64_next(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
VMFA_HD uint64_t key2(uint64_t a, uint64_t b) {
  uint64_t s = a;
  const uint64_t h = sm64_next(s);
  s ^= b + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
  return sm64_next(s);
}
VMFA_HD uint64_t key3(uint64_t a, uint64_t b, uint64_t c) { return key2(key2(a, b), c); }

VMFA_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

// uniform_component (rng.hpp:91-98)
VMFA_HD int extra_candidate(uint64_t seed, uint64_t iteration, uint64_t n, int C) {
  return static_cast<int>(mulhi64(key3(seed, iteration, n), static_cast<uint64_t>(C)));
}

// xoshiro256++ stream seeded through splitmix64 (rng.hpp:30-86), host only.
struct HostStream {
  uint64_t w[4];
  double spare = 0.0;
  bool has_spare = false;
  explicit HostStream(uint64_t seed) {
    uint64_t s = seed;
    for (auto& x : w) x = sm64_next(s);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t out = rotl(w[0] + w[3], 23) + w[0];
    const uint64_t t = w[1] << 17;
    w[2] ^= w[0];
    w[3] ^= w[1];
    w[1] ^= w[2];
    w[0] ^= w[3];
    w[2] ^= t;
    w[3] = rotl(w[3], 45);
    return out;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  int64_t uniform_int(int64_t bound) { return static_cast<int64_t>(mulhi64(next(), static_cast<uint64_t>(bound))); }
  double gaussian() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586 * u2;
    spare = r * std::sin(a);
    has_spare = true;
    return r * std::cos(a);
  }
};

}  // namespace vmfa_b200
