// rng.cu -- device RNG entry points: per-key sequential draws (parity
// checks of philox.cuh against the reference stream, rng.hpp:77-134) and
// batched key derivation (the RngKey tree, rng.hpp:58-66).
#include "fnb_common.cuh"
#include "philox.cuh"
#include "glibc_math.cuh"

namespace fnb {

// kind 0: next_u64, 1: uniform (as bits), 2: below(n), 3: normal(0, 1) (as
// bits; rng.hpp:111-116 with the glibc-exact log / cos of glibc_math.cuh)
__global__ void k_stream_draws(const uint32_t* __restrict__ keys, int n_keys, int n_draws, int kind, uint64_t n,
                               uint64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_keys) return;
  Stream s(Key4{{keys[4 * i], keys[4 * i + 1], keys[4 * i + 2], keys[4 * i + 3]}});
  for (int d = 0; d < n_draws; ++d) {
    uint64_t v;
    if (kind == 0) v = s.next_u64();
    else if (kind == 1) v = uint64_t(__double_as_longlong(s.uniform()));
    else if (kind == 2) v = s.below(n);
    else {
      const double a0 = s.uniform();
      const double a1 = s.uniform();
      v = uint64_t(__double_as_longlong(glibc::normal_from_uniforms(a0, a1, 0.0, 1.0)));
    }
    out[size_t(i) * n_draws + d] = v;
  }
}

// out[i] = parent.split(base + i)
__global__ void k_split_keys(Key4 parent, uint64_t base, int n, uint32_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Key4 k = key_split(parent, base + uint64_t(i));
  *reinterpret_cast<uint4*>(out + 4 * size_t(i)) = make_uint4(k.w[0], k.w[1], k.w[2], k.w[3]);
}

cudaError_t launch_stream_draws(const uint32_t* keys, int n_keys, int n_draws, int kind, uint64_t n, uint64_t* out,
                                cudaStream_t st) {
  if (n_keys <= 0) return cudaSuccess;
  k_stream_draws<<<(n_keys + 127) / 128, 128, 0, st>>>(keys, n_keys, n_draws, kind, n, out);
  return cudaGetLastError();
}

cudaError_t launch_split_keys(const uint32_t parent[4], uint64_t base, int n, uint32_t* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const Key4 k{{parent[0], parent[1], parent[2], parent[3]}};
  k_split_keys<<<(n + 255) / 256, 256, 0, st>>>(k, base, n, out);
  return cudaGetLastError();
}

}  // namespace fnb
