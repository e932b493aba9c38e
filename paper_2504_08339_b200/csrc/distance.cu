// distance.cu -- K3: compatibility distance of every genome against S
// species representatives (distance, ops.hpp:415-473), FP64, bit-exact.
//
// The reference walks g1's rows in row order, looks each marker up in g2 by
// linear scan and accumulates the attribute differences sequentially.  Here:
//   * each representative gets an open-addressing marker table once
//     (k_rep_tables), so every lookup is ~1 probe instead of an O(C) scan;
//   * rows in chunks of 32 (one per lane, coalesced): each lane computes its
//     row's term against every representative into a shared tile, then lane
//     s adds the chunk in row order -- the reference's sequential FP64 sum
//     with separately rounded ops, bit for bit (distance_warp.cuh).
#include <algorithm>

#include "distance_warp.cuh"

namespace fnb {

// Bloom filter words per representative (log2): about 16 bits per connection
// key (false positives ~6%), within a 24 KB shared-memory budget for S reps
// (the rest of the SM's shared memory keeps the warps in flight).
__host__ inline int filter_words_log2(int S, int C) {
  int lg = 5;  // 32 words = 1024 bits minimum
  while (lg < 11 && (size_t(1) << (lg + 5)) < size_t(16) * C) ++lg;
  while (lg > 5 && size_t(S) * (size_t(4) << lg) > 24 * 1024) --lg;
  return lg;
}

__host__ inline size_t rep_tables_bytes(int S, int N, int C) {
  const size_t hn = size_t(table_capacity(N)), hc = size_t(table_capacity(C));
  return size_t(S) * (hn * 12 + hc * 20 + 8 + (size_t(4) << filter_words_log2(S, C))) + 64;
}

// one CTA per representative: marker tables + the connection-key filter
__global__ void k_rep_tables(const double* __restrict__ rn, const double* __restrict__ rc, int N, int C,
                             RepTables t, uint32_t* filt) {
  const int s = blockIdx.x;
  uint32_t* f = filt + (size_t(s) << t.fw_log2);
  for (int i = threadIdx.x; i < (1 << t.fw_log2); i += blockDim.x) f[i] = 0u;
  __syncthreads();
  const double* cr = rc + size_t(s) * C * kConnCols;
  for (int r = threadIdx.x; r < C; r += blockDim.x) {
    const double in = cr[r * kConnCols + kIn];
    if (isnan(in)) continue;
    const uint32_t b = filter_bit(conn_key(in, cr[r * kConnCols + kOut]), t.fw_log2);
    atomicOr(&f[b >> 5], 1u << (b & 31));
  }
  rep_table_build(rn + size_t(s) * N * kNodeCols, cr, N, C, t.nkeys + size_t(s) * t.Hn, t.nrows + size_t(s) * t.Hn,
                  t.Hn, t.ckeys + size_t(s) * t.Hc, t.crows + size_t(s) * t.Hc, t.cw + size_t(s) * t.Hc, t.Hc,
                  t.counts + 2 * s);
}

// persistent CTAs, one warp per genome; the representatives' filters are
// copied to shared memory once per CTA, so a connection key absent from a
// representative (most lookups: disjoint genes, other species) is settled
// by one shared-memory bit test instead of an L1/L2 probe sequence
__global__ void __launch_bounds__(256)
k_distance(const double* __restrict__ nodes, const double* __restrict__ conns, int P,
           const double* __restrict__ rn, const double* __restrict__ rc, int S, RepTables t, int N, int C,
           double cd, double ch, double* __restrict__ out, const int* __restrict__ only_unassigned,
           const int* __restrict__ after_founder) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5;
  uint32_t* sf = reinterpret_cast<uint32_t*>(smem_raw);
  const int fw = S << t.fw_log2;
  for (int i = threadIdx.x; i < fw; i += blockDim.x) sf[i] = t.filt[i];
  __syncthreads();
  RepTables ts = t;
  ts.filt = sf;
  double* tile = reinterpret_cast<double*>(smem_raw + size_t(fw) * 4) + size_t(warp) * S * 33;
  for (int g = blockIdx.x * warps + warp; g < P; g += gridDim.x * warps) {
    // speciation rounds only need genomes still without a species (and, for
    // a founding round, after the founder): skip the rest without touching HBM
    if (only_unassigned && only_unassigned[g] >= 0) continue;
    if (after_founder && (after_founder[0] < 0 || g <= after_founder[0])) continue;
    distance_warp(nodes + size_t(g) * N * kNodeCols, conns + size_t(g) * C * kConnCols, rn, rc, S, ts, N, C, cd, ch,
                  tile, out + size_t(g) * S);
  }
}

// ---- host launcher -----------------------------------------------------------
cudaError_t launch_distance_masked(const double* nodes, const double* conns, int P, const double* rn,
                                   const double* rc, int S, int N, int C, double cd, double ch, double* out,
                                   void* scratch, size_t scratch_bytes, const int* only_unassigned,
                                   const int* after_founder, cudaStream_t st);

cudaError_t launch_distance(const double* nodes, const double* conns, int P, const double* rn, const double* rc,
                            int S, int N, int C, double cd, double ch, double* out, void* scratch,
                            size_t scratch_bytes, cudaStream_t st) {
  return launch_distance_masked(nodes, conns, P, rn, rc, S, N, C, cd, ch, out, scratch, scratch_bytes, nullptr,
                                nullptr, st);
}

cudaError_t launch_distance_masked(const double* nodes, const double* conns, int P, const double* rn,
                                   const double* rc, int S, int N, int C, double cd, double ch, double* out,
                                   void* scratch, size_t scratch_bytes, const int* only_unassigned,
                                   const int* after_founder, cudaStream_t st) {
  if (S <= 0 || P <= 0) return cudaSuccess;
  RepTables t;
  t.Hn = table_capacity(N);
  t.Hc = table_capacity(C);
  uint8_t* p = static_cast<uint8_t*>(scratch);
  t.nkeys = reinterpret_cast<unsigned long long*>(p); p += size_t(S) * t.Hn * 8;
  t.ckeys = reinterpret_cast<unsigned long long*>(p); p += size_t(S) * t.Hc * 8;
  t.nrows = reinterpret_cast<int*>(p); p += size_t(S) * t.Hn * 4;
  t.cw = reinterpret_cast<double*>(p); p += size_t(S) * t.Hc * 8;
  t.crows = reinterpret_cast<int*>(p); p += size_t(S) * t.Hc * 4;
  t.counts = reinterpret_cast<int*>(p); p += size_t(S) * 8;
  t.fw_log2 = filter_words_log2(S, C);
  uint32_t* filt = reinterpret_cast<uint32_t*>(p); p += size_t(S) * (size_t(4) << t.fw_log2);
  t.filt = filt;
  if (size_t(p - static_cast<uint8_t*>(scratch)) > scratch_bytes) return cudaErrorInvalidValue;
  k_rep_tables<<<S, 256, 0, st>>>(rn, rc, N, C, t, filt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int warps = 8;
  const size_t smem = (size_t(S) << t.fw_log2) * 4 + size_t(warps) * S * 33 * sizeof(double);
  e = cudaFuncSetAttribute(k_distance, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;  // persistent grid: the co-resident CTAs
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_distance, 32 * warps, smem);
  if (e != cudaSuccess) return e;
  const int grid = std::max(1, std::min((P + warps - 1) / warps, std::max(1, per_sm) * sms));
  k_distance<<<grid, 32 * warps, smem, st>>>(nodes, conns, P, rn, rc, S, t, N, C, cd, ch, out, only_unassigned,
                                             after_founder);
  return cudaGetLastError();
}

size_t distance_scratch_bytes(int S, int N, int C) { return rep_tables_bytes(S, N, C); }

}  // namespace fnb
