// Device edge-membership table: undirected edge {a, b} -> one 32-byte bucket
// probe (a single HBM/L2 sector) instead of a dependent binary search over an
// adjacency list. Buckets hold 4 u64 keys (min << 32 | max); first-fit
// two-choice insertion (bucket h1, else h2) means a key lives in h2 only if h1
// was already full when it was inserted — and buckets never empty again — so a
// lookup reads h2 only when h1 is full. Load factor <= 1/2.
//
// Membership in a bound-restricted in-list N(b) ∩ [lo, hi) equals edge
// existence for any a already inside [lo, hi) (the driver range is), and
// out-lists are whole lists, so every "other list" test of an eager step
// (walker.hpp:39-55) is one lookup.
#pragma once

#include <cstdint>

#include "rng.cuh"

namespace agpm_b200 {

constexpr unsigned long long kEmptyKey = ~0ull;
constexpr unsigned long long kHash2Salt = 0x5851f42d4c957f2dull;

__device__ __forceinline__ bool edge_lookup(const unsigned long long* __restrict__ table, uint32_t mask,
                                            uint32_t a, uint32_t b) {
  const unsigned long long key = a < b ? ((unsigned long long)a << 32) | b : ((unsigned long long)b << 32) | a;
  const unsigned long long h = mix64(key);
  const ulonglong2* bk = reinterpret_cast<const ulonglong2*>(table + 4ull * (h & mask));
  ulonglong2 x = __ldg(bk), y = __ldg(bk + 1);
  if (x.x == key || x.y == key || y.x == key || y.y == key) return true;
  if (y.y == kEmptyKey) return false;  // h1 not full: the key was never pushed to h2
  const unsigned long long h2 = mix64(key ^ kHash2Salt);
  bk = reinterpret_cast<const ulonglong2*>(table + 4ull * (h2 & mask));
  x = __ldg(bk);
  y = __ldg(bk + 1);
  return x.x == key || x.y == key || y.x == key || y.y == key;
}

}  // namespace agpm_b200
