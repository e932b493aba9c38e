// crossover.cu -- K5: population-wide crossover by historical-marker
// alignment (crossover, ops.hpp:382-407), bit-exact.
//
// One warp per child.  The reference copies the fit parent, then walks its
// node rows and connection rows in order, finds each marker in the other
// parent by linear scan and flips one fair coin per attribute of every
// matched gene from ONE sequential RngStream(key).  Here the other parent's
// markers go into a per-warp shared-memory table (~1 probe per lookup) and,
// because Philox is counter based, every lane computes the stream position
// of its own rows' coins from a ballot prefix count of matched rows -- node
// gene k consumes draws 4k..4k+3 (attributes 1..4), connection gene k draw
// 4*M_nodes + k -- so the whole child is produced in one parallel pass.
// coin(0.5) is uniform() < 0.5, i.e. the top bit of the u64 draw is 0.
#include "fnb_common.cuh"
#include "keytable.cuh"
#include "philox.cuh"

namespace fnb {

__device__ __forceinline__ bool coin_half(uint64_t x) { return (x >> 63) == 0; }

__global__ void __launch_bounds__(128)
k_crossover(const double* __restrict__ nodes, const double* __restrict__ conns, const int32_t* __restrict__ fit_idx,
            const int32_t* __restrict__ oth_idx, const uint32_t* __restrict__ keys, int n_children, int N, int C,
            double* __restrict__ child_nodes, double* __restrict__ child_conns, size_t smem_per_warp) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= n_children) return;
  const int Hn = table_capacity(N), Hc = table_capacity(C);
  uint8_t* base = smem_raw + size_t(warp) * smem_per_warp;
  unsigned long long* nk = reinterpret_cast<unsigned long long*>(base);
  unsigned long long* ck = nk + Hn;
  int* nr = reinterpret_cast<int*>(ck + Hc);
  int* cr = nr + Hn;

  const int fi = fit_idx[c], oi = oth_idx[c];
  const double* fn = nodes + size_t(fi) * N * kNodeCols;
  const double* fc = conns + size_t(fi) * C * kConnCols;
  const double* on = nodes + size_t(oi) * N * kNodeCols;
  const double* oc = conns + size_t(oi) * C * kConnCols;
  double* cn = child_nodes + size_t(c) * N * kNodeCols;
  double* cc = child_conns + size_t(c) * C * kConnCols;
  const Key4 key{{keys[4 * c], keys[4 * c + 1], keys[4 * c + 2], keys[4 * c + 3]}};

  // marker tables of the other parent
  for (int i = lane; i < Hn; i += 32) { nk[i] = kEmptyKey; nr[i] = 0x7fffffff; }
  for (int i = lane; i < Hc; i += 32) { ck[i] = kEmptyKey; cr[i] = 0x7fffffff; }
  __syncwarp();
  for (int r = lane; r < N; r += 32) {
    const double k = on[r * kNodeCols + kKey];
    if (!isnan(k)) table_insert(nk, nr, Hn - 1, node_key(k), r);
  }
  for (int r = lane; r < C; r += 32) {
    const double2 a = *reinterpret_cast<const double2*>(oc + r * kConnCols);
    if (!isnan(a.x)) table_insert(ck, cr, Hc - 1, conn_key(a.x, a.y), r);
  }
  __syncwarp();

  // node genes: 4 coins each (attributes 1..4), ops.hpp:388-396
  int matched_before = 0;
  for (int r0 = 0; r0 < N; r0 += 32) {
    const int r = r0 + lane;
    double row[kNodeCols];
    int m = -1;
    if (r < N) {
#pragma unroll
      for (int a = 0; a < kNodeCols; ++a) row[a] = fn[r * kNodeCols + a];
      if (!isnan(row[kKey])) m = table_find(nk, nr, Hn - 1, node_key(row[kKey]));
    }
    const unsigned bal = __ballot_sync(0xffffffffu, m >= 0);
    if (m >= 0) {
      const uint64_t q = 4ull * uint64_t(matched_before + __popc(bal & ((1u << lane) - 1u)));
      uint32_t b0[4], b1[4];
      stream_block(key, q >> 1, b0);        // draws q, q+1
      stream_block(key, (q >> 1) + 1, b1);  // draws q+2, q+3
      const uint64_t d[4] = {(uint64_t(b0[3]) << 32) | b0[2], (uint64_t(b0[1]) << 32) | b0[0],
                             (uint64_t(b1[3]) << 32) | b1[2], (uint64_t(b1[1]) << 32) | b1[0]};
      const double* theirs = on + m * kNodeCols;
#pragma unroll
      for (int a = 1; a < kNodeCols; ++a)
        if (coin_half(d[a - 1])) row[a] = theirs[a];
    }
    if (r < N) {
#pragma unroll
      for (int a = 0; a < kNodeCols; ++a) cn[r * kNodeCols + a] = row[a];
    }
    matched_before += __popc(bal);
  }
  // connection genes: 1 coin each (weight), ops.hpp:397-405
  const uint64_t q0 = 4ull * uint64_t(matched_before);
  int cmatched = 0;
  for (int r0 = 0; r0 < C; r0 += 32) {
    const int r = r0 + lane;
    double2 a = make_double2(__longlong_as_double(0x7ff8000000000000ll), 0.0), b = make_double2(0.0, 0.0);
    int m = -1;
    if (r < C) {
      a = *reinterpret_cast<const double2*>(fc + r * kConnCols);
      b = *reinterpret_cast<const double2*>(fc + r * kConnCols + 2);
      if (!isnan(a.x)) m = table_find(ck, cr, Hc - 1, conn_key(a.x, a.y));
    }
    const unsigned bal = __ballot_sync(0xffffffffu, m >= 0);
    if (m >= 0) {
      const uint64_t q = q0 + uint64_t(cmatched + __popc(bal & ((1u << lane) - 1u)));
      if (coin_half(stream_u64_at(key, q))) b.y = oc[m * kConnCols + kW];
    }
    if (r < C) {
      *reinterpret_cast<double2*>(cc + r * kConnCols) = a;
      *reinterpret_cast<double2*>(cc + r * kConnCols + 2) = b;
    }
    cmatched += __popc(bal);
  }
}

size_t crossover_smem_per_warp(int N, int C) {
  return align16(size_t(table_capacity(N) + table_capacity(C)) * 12);
}

cudaError_t launch_crossover(const double* nodes, const double* conns, const int32_t* fit, const int32_t* oth,
                             const uint32_t* keys, int n, int N, int C, double* cn, double* cc, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const size_t per_warp = crossover_smem_per_warp(N, C);
  int warps = 4;
  while (warps > 1 && per_warp * warps > 96 * 1024) warps >>= 1;
  const size_t smem = per_warp * warps;
  cudaError_t e = cudaFuncSetAttribute(k_crossover, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k_crossover<<<(n + warps - 1) / warps, 32 * warps, smem, st>>>(nodes, conns, fit, oth, keys, n, N, C, cn, cc,
                                                                 per_warp);
  return cudaGetLastError();
}

}  // namespace fnb
