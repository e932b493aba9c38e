// crossover.cu -- K5: population-wide crossover by historical-marker
// alignment (crossover, ops.hpp:382-407), bit-exact.
//
// One 128-thread CTA per child.  The reference copies the fit parent, then walks its
// node rows and connection rows in order, finds each marker in the other
// parent by linear scan and flips one fair coin per attribute of every
// matched gene from ONE sequential RngStream(key).  Here the other parent's
// markers go into a per-CTA shared-memory table (~1 probe per lookup) and,
// because Philox is counter based, every thread computes the stream position
// of its own rows' coins from a block prefix count of matched rows -- node
// gene k consumes draws 4k..4k+3 (attributes 1..4), connection gene k draw
// 4*M_nodes + k -- so the whole child is produced in one parallel pass.
// coin(0.5) is uniform() < 0.5, i.e. the top bit of the u64 draw is 0.
#include "fnb_common.cuh"
#include "keytable.cuh"
#include "philox.cuh"

namespace fnb {

__device__ __forceinline__ bool coin_half(uint64_t x) { return (x >> 63) == 0; }

constexpr int kXWarps = 4;  // one 128-thread CTA per child

// Block-wide exclusive prefix of `flag` over the CTA's threads (thread order =
// row order within a chunk) and the chunk total.  Two barriers.
__device__ __forceinline__ int block_prefix(bool flag, int* s_cnt, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, flag);
  if (lane == 0) s_cnt[warp] = __popc(bal);
  __syncthreads();
  int before = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < kXWarps; ++w) {
    const int c = s_cnt[w];
    before += w < warp ? c : 0;
    total += c;
  }
  __syncthreads();  // s_cnt is reused by the next chunk
  return before + __popc(bal & ((1u << lane) - 1u));
}

__global__ void __launch_bounds__(kXWarps * 32)
k_crossover(const double* __restrict__ nodes, const double* __restrict__ conns, const int32_t* __restrict__ fit_idx,
            const int32_t* __restrict__ oth_idx, const uint32_t* __restrict__ keys, int n_children, int N, int C,
            double* __restrict__ child_nodes, double* __restrict__ child_conns) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ int s_cnt[kXWarps];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int c = blockIdx.x;
  if (c >= n_children) return;
  const int Hn = table_capacity(N), Hc = table_capacity(C);
  unsigned long long* nk = reinterpret_cast<unsigned long long*>(smem_raw);
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

  // the fit parent's first node chunk is loaded before the table build
  double row0[kNodeCols];
  if (tid < N) {
#pragma unroll
    for (int a = 0; a < kNodeCols; ++a) row0[a] = fn[tid * kNodeCols + a];
  }

  // marker tables of the other parent
  for (int i = tid; i < Hn; i += nt) { nk[i] = kEmptyKey; nr[i] = 0x7fffffff; }
  for (int i = tid; i < Hc; i += nt) { ck[i] = kEmptyKey; cr[i] = 0x7fffffff; }
  __syncthreads();
  for (int r = tid; r < N; r += nt) {
    const double k = on[r * kNodeCols + kKey];
    if (!isnan(k)) table_insert(nk, nr, Hn - 1, node_key(k), r);
  }
  {
    double2 na = tid < C ? *reinterpret_cast<const double2*>(oc + tid * kConnCols) : make_double2(0.0, 0.0);
    for (int r = tid; r < C; r += nt) {
      const double2 a = na;  // the next chunk's markers are in flight during this chunk's inserts
      if (r + nt < C) na = *reinterpret_cast<const double2*>(oc + (r + nt) * kConnCols);
      if (!isnan(a.x)) table_insert(ck, cr, Hc - 1, conn_key(a.x, a.y), r);
    }
  }
  __syncthreads();

  // node genes: 4 coins each (attributes 1..4), ops.hpp:388-396
  int matched_before = 0;
  for (int r0 = 0; r0 < N; r0 += nt) {
    const int r = r0 + tid;
    double row[kNodeCols];
    int m = -1;
    if (r < N) {
#pragma unroll
      for (int a = 0; a < kNodeCols; ++a) row[a] = r0 == 0 ? row0[a] : fn[r * kNodeCols + a];
      if (!isnan(row[kKey])) m = table_find(nk, nr, Hn - 1, node_key(row[kKey]));
    }
    int total;
    const int rank = block_prefix(m >= 0, s_cnt, total);
    if (m >= 0) {
      const uint64_t q = 4ull * uint64_t(matched_before + rank);
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
    matched_before += total;
  }
  // connection genes: 1 coin each (weight), ops.hpp:397-405
  const uint64_t q0 = 4ull * uint64_t(matched_before);
  int cmatched = 0;
  // the next chunk's fit rows are loaded before this chunk's barriers
  const double2 kNone = make_double2(__longlong_as_double(0x7ff8000000000000ll), 0.0);
  double2 na = kNone, nb = make_double2(0.0, 0.0);
  if (tid < C) {
    na = *reinterpret_cast<const double2*>(fc + tid * kConnCols);
    nb = *reinterpret_cast<const double2*>(fc + tid * kConnCols + 2);
  }
  for (int r0 = 0; r0 < C; r0 += nt) {
    const int r = r0 + tid;
    double2 a = na, b = nb;
    if (r + nt < C) {
      na = *reinterpret_cast<const double2*>(fc + (r + nt) * kConnCols);
      nb = *reinterpret_cast<const double2*>(fc + (r + nt) * kConnCols + 2);
    }
    int m = -1;
    if (r < C && !isnan(a.x)) m = table_find(ck, cr, Hc - 1, conn_key(a.x, a.y));
    int total;
    const int rank = block_prefix(m >= 0, s_cnt, total);
    if (m >= 0) {
      const uint64_t q = q0 + uint64_t(cmatched + rank);
      if (coin_half(stream_u64_at(key, q))) b.y = oc[m * kConnCols + kW];
    }
    if (r < C) {
      *reinterpret_cast<double2*>(cc + r * kConnCols) = a;
      *reinterpret_cast<double2*>(cc + r * kConnCols + 2) = b;
    }
    cmatched += total;
  }
}

size_t crossover_smem(int N, int C) { return align16(size_t(table_capacity(N) + table_capacity(C)) * 12); }

cudaError_t launch_crossover(const double* nodes, const double* conns, const int32_t* fit, const int32_t* oth,
                             const uint32_t* keys, int n, int N, int C, double* cn, double* cc, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = crossover_smem(N, C);
  cudaError_t e = cudaFuncSetAttribute(k_crossover, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k_crossover<<<n, kXWarps * 32, smem, st>>>(nodes, conns, fit, oth, keys, n, N, C, cn, cc);
  return cudaGetLastError();
}

}  // namespace fnb
