// keytable.cuh -- open-addressing key -> first-row tables for historical
// marker alignment.  Replaces the reference's O(N) / O(C) linear scans
// find_node / find_conn (genome.hpp:195-210) with ~1 probe: a node key or a
// connection (in, out) pair maps to the LOWEST row holding it, which is what
// the reference's first-match scan returns when a corrupt genome repeats a
// key.  Keys are 64-bit: node = uint32(key), conn = uint32(in) << 32 |
// uint32(out); ~0 marks an empty slot (a pair (-1,-1) cannot be stored --
// negative keys are invalid genomes, genome.hpp:373).
#pragma once
#include <cstdint>

namespace fnb {

constexpr unsigned long long kEmptyKey = ~0ull;

__host__ __device__ __forceinline__ uint32_t hash_key(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return uint32_t(k);
}

__host__ __device__ __forceinline__ unsigned long long conn_key(double in, double out) {
  return (static_cast<unsigned long long>(static_cast<uint32_t>(int(in))) << 32) |
         static_cast<uint32_t>(int(out));
}
__host__ __device__ __forceinline__ unsigned long long node_key(double key) {
  return static_cast<uint32_t>(int(key));
}

__host__ __device__ inline int table_capacity(int n) {
  int h = 16;
  while (h < 2 * n) h <<= 1;
  return h;
}

// Insert (parallel-safe): claim a slot for the key, keep the minimum row.
__device__ __forceinline__ void table_insert(unsigned long long* keys, int* rows, int mask,
                                             unsigned long long key, int row) {
  uint32_t s = hash_key(key) & uint32_t(mask);
  for (;;) {
    const unsigned long long prev = atomicCAS(&keys[s], kEmptyKey, key);
    if (prev == kEmptyKey || prev == key) {
      atomicMin(&rows[s], row);
      return;
    }
    s = (s + 1) & uint32_t(mask);
  }
}

__device__ __forceinline__ int table_find(const unsigned long long* keys, const int* rows, int mask,
                                          unsigned long long key) {
  uint32_t s = hash_key(key) & uint32_t(mask);
  for (;;) {
    const unsigned long long k = keys[s];
    if (k == key) return rows[s];
    if (k == kEmptyKey) return -1;
    s = (s + 1) & uint32_t(mask);
  }
}

}  // namespace fnb
