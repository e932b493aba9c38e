// philox.cuh -- bit-exact device restatement of the reference RNG
// (rng.hpp:19-134): Philox4x32-10, the RngKey tree and RngStream.
//
// Because Philox is counter based, stream draw q of a key is a pure function
// of (key, q): draw q comes from block q/2 of the stream, high half first
// (rng.hpp:81-87: avail counts down 4 -> 2 -> 0, so the first u64 of a block
// is words 2,3 and the second words 0,1).  Kernels use this to give every
// lane its own slice of one sequential stream without replaying it.
#pragma once
#include <cstdint>

namespace fnb {

struct Key4 {
  uint32_t w[4];
};

__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
#ifdef __CUDA_ARCH__
    const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
    const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
#else
    const uint64_t p0 = uint64_t(0xD2511F53u) * c[0], p1 = uint64_t(0xCD9E8D57u) * c[2];
    const uint32_t lo0 = uint32_t(p0), hi0 = uint32_t(p0 >> 32), lo1 = uint32_t(p1), hi1 = uint32_t(p1 >> 32);
#endif
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// RngKey(seed) (rng.hpp:48-56)
__host__ __device__ __forceinline__ Key4 key_from_seed(uint64_t seed) {
  Key4 k{{uint32_t(seed), uint32_t(seed >> 32), 0x464C4154u, 0x4E454154u}};
  philox4x32_10(k.w, 0x243F6A88u, 0x85A308D3u);
  return k;
}

// RngKey::split (rng.hpp:58-66)
__host__ __device__ __forceinline__ Key4 key_split(const Key4& k, uint64_t index) {
  Key4 c{{uint32_t(index), uint32_t(index >> 32), k.w[2], k.w[3]}};
  philox4x32_10(c.w, k.w[0], k.w[1]);
  return c;
}

// Block b of RngStream(k) (refill, rng.hpp:119-128)
__host__ __device__ __forceinline__ void stream_block(const Key4& k, uint64_t b, uint32_t out[4]) {
  out[0] = uint32_t(b);
  out[1] = uint32_t(b >> 32);
  out[2] = k.w[2] ^ 0x9E3779B9u;
  out[3] = k.w[3];
  philox4x32_10(out, k.w[0], k.w[1]);
}

// Draw q (0-based) of RngStream(k).next_u64()
__host__ __device__ __forceinline__ uint64_t stream_u64_at(const Key4& k, uint64_t q) {
  uint32_t b[4];
  stream_block(k, q >> 1, b);
  return (q & 1) ? ((uint64_t(b[1]) << 32) | b[0]) : ((uint64_t(b[3]) << 32) | b[2]);
}

// uniform() = (u64 >> 11) * 2^-53 (rng.hpp:90-92); coin(p) = uniform < p
__host__ __device__ __forceinline__ double u64_to_uniform(uint64_t x) { return double(x >> 11) * 0x1.0p-53; }

// Sequential stream with a one-block buffer (rng.hpp:77-134).  The block is
// kept as its two u64 halves so no array is indexed dynamically (registers,
// not local memory, on the device).
struct Stream {
  Key4 key;
  uint64_t block;
  uint64_t first, second;  // draw order within the current block
  int avail;               // u32 words left, as in the reference (4, 2, 0)
  __host__ __device__ explicit Stream(const Key4& k) : key(k), block(0), first(0), second(0), avail(0) {}
  __host__ __device__ __forceinline__ uint64_t next_u64() {
    if (avail == 0) {
      uint32_t b[4];
      stream_block(key, block, b);
      ++block;
      first = (uint64_t(b[3]) << 32) | b[2];
      second = (uint64_t(b[1]) << 32) | b[0];
      avail = 4;
    }
    avail -= 2;
    return avail == 2 ? first : second;
  }
  __host__ __device__ __forceinline__ double uniform() { return u64_to_uniform(next_u64()); }
  __host__ __device__ __forceinline__ bool coin(double p) { return uniform() < p; }
  // below(n) (rng.hpp:99-106): rejection of the top partial range
  __host__ __device__ __forceinline__ uint64_t below(uint64_t n) {
    const uint64_t mx = ~uint64_t(0);
    const uint64_t limit = mx - ((mx % n) + 1) % n;
    uint64_t x = next_u64();
    while (x > limit) x = next_u64();
    return x % n;
  }
  __host__ __device__ __forceinline__ int index(int n) { return int(below(uint64_t(n))); }
  // below(n) with the rejection limit computed once by the caller (the same n
  // drawn repeatedly: the 64-bit remainders of the limit are most of the cost)
  __host__ __device__ __forceinline__ static uint64_t below_limit(uint64_t n) {
    const uint64_t mx = ~uint64_t(0);
    return mx - ((mx % n) + 1) % n;
  }
  __host__ __device__ __forceinline__ int index_lim(int n, uint64_t limit) {
    uint64_t x = next_u64();
    while (x > limit) x = next_u64();
    return int(x % uint64_t(n));
  }
  // draws consumed so far
  __host__ __device__ __forceinline__ uint64_t position() const { return block * 2 - uint64_t(avail / 2); }
};

}  // namespace fnb
