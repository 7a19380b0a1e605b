// Counter RNG shared by host and device code. Bit-for-bit the reference's
// CounterRng (rng.hpp:10-56): a SplitMix64-finaliser hash keyed by
// (seed, stream1, stream2), Lemire bounded draws. The sampler's per-sample
// stream is CounterRng(seed, 0, sample_id) — the reference's single-worker
// stream (ns_engine.cpp:72) — so every device sample id reproduces the
// reference's draw exactly.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define AGPM_HD __host__ __device__ __forceinline__
#else
#define AGPM_HD inline
#endif

namespace agpm_b200 {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
constexpr uint64_t kMixA = 0xbf58476d1ce4e5b9ull;
constexpr uint64_t kMixB = 0x94d049bb133111ebull;
constexpr uint64_t kColorTag = 0x636f6c6f72ull;  // "color", rng.hpp:68

AGPM_HD uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= kMixA;
  z ^= z >> 27;
  z *= kMixB;
  z ^= z >> 31;
  return z;
}

AGPM_HD uint64_t derive_key(uint64_t seed, uint64_t s1, uint64_t s2) {
  uint64_t h = mix64(seed + kGolden);
  h = mix64(h ^ (s1 + kMixA));
  h = mix64(h ^ (s2 + kMixB));
  return h;
}

AGPM_HD uint64_t mul_hi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

struct CounterRng {
  uint64_t key;
  uint64_t ctr;
  AGPM_HD explicit CounterRng(uint64_t seed, uint64_t s1 = 0, uint64_t s2 = 0)
      : key(derive_key(seed, s1, s2)), ctr(0) {}
  AGPM_HD uint64_t next_u64() {
    ctr += kGolden;
    return mix64(key ^ ctr);
  }
  AGPM_HD double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  // uniform in [0, n), n >= 1; same rejection rule and draw count as rng.hpp:40-51
  AGPM_HD uint64_t next_below(uint64_t n) {
    uint64_t x = next_u64();
    uint64_t lo = x * n;
    uint64_t hi = mul_hi64(x, n);
    if (lo < n) {
      uint64_t t = (0 - n) % n;
      while (lo < t) {
        x = next_u64();
        lo = x * n;
        hi = mul_hi64(x, n);
      }
    }
    return hi;
  }
};

// Philox4x32-10 (Salmon et al., SC'11: 10 rounds of two 32x32->64 multiplies,
// Weyl key schedule). The optional sampler stream of the north star: sample i
// of seed s draws u64 number t from one block with counter (t, i) and key s —
// a pure function of (seed, sample id, draw index), like CounterRng, but not
// the reference's stream (so parity for it is against the oracle restatement,
// oracle/agpm_oracle.c, and statistics; the reference-parity policy stays
// CounterRng).
AGPM_HD void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c[0];
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c[2];
    const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c[3] ^ k1;
    c[1] = static_cast<uint32_t>(p1);
    c[3] = static_cast<uint32_t>(p0);
    c[0] = n0;
    c[2] = n2;
  }
}

struct PhiloxRng {
  uint64_t key;  // seed
  uint64_t ctr;  // draws taken
  uint64_t id;   // sample id
  AGPM_HD explicit PhiloxRng(uint64_t seed, uint64_t s1 = 0, uint64_t s2 = 0) : key(seed), ctr(0), id(s2) {
    (void)s1;  // single-stream-family policy: the worker index is not part of the counter
  }
  AGPM_HD uint64_t next_u64() {
    uint32_t c[4] = {static_cast<uint32_t>(ctr), static_cast<uint32_t>(ctr >> 32), static_cast<uint32_t>(id),
                     static_cast<uint32_t>(id >> 32)};
    ++ctr;
    philox4x32_10(c, static_cast<uint32_t>(key), static_cast<uint32_t>(key >> 32));
    return static_cast<uint64_t>(c[0]) | (static_cast<uint64_t>(c[1]) << 32);
  }
  // same Lemire rule as CounterRng::next_below
  AGPM_HD uint64_t next_below(uint64_t n) {
    uint64_t x = next_u64();
    uint64_t lo = x * n;
    uint64_t hi = mul_hi64(x, n);
    if (lo < n) {
      uint64_t t = (0 - n) % n;
      while (lo < t) {
        x = next_u64();
        lo = x * n;
        hi = mul_hi64(x, n);
      }
    }
    return hi;
  }
};

// rng.hpp:60-65
AGPM_HD bool edge_keep_decision(uint64_t seed, uint32_t u, uint32_t v, double p) {
  uint32_t a = u < v ? u : v;
  uint32_t b = u < v ? v : u;
  uint64_t h = derive_key(seed, a, b);
  return static_cast<double>(h >> 11) * 0x1.0p-53 < p;
}

// rng.hpp:67-70
AGPM_HD uint32_t vertex_color_decision(uint64_t seed, uint32_t v, uint32_t c) {
  uint64_t h = derive_key(seed, v, kColorTag);
  return static_cast<uint32_t>(mul_hi64(h, c));
}

}  // namespace agpm_b200
