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
#include "distance_warp.cuh"

namespace fnb {

__host__ inline size_t rep_tables_bytes(int S, int N, int C) { return size_t(S) * rep_table_bytes_one(N, C) + 64; }

// one CTA per representative
__global__ void k_rep_tables(const double* __restrict__ rn, const double* __restrict__ rc, int N, int C,
                             RepTables t) {
  const int s = blockIdx.x;
  rep_table_build(rn + size_t(s) * N * kNodeCols, rc + size_t(s) * C * kConnCols, N, C, t.n + size_t(s) * t.Hn, t.Hn,
                  t.c + size_t(s) * t.Hc, t.crow + size_t(s) * t.Hc, t.Hc, t.counts + 2 * s);
}

// one warp per genome
__global__ void __launch_bounds__(128)
k_distance(const double* __restrict__ nodes, const double* __restrict__ conns, int P,
           const double* __restrict__ rn, const double* __restrict__ rc, int S, RepTables t, int N, int C,
           double cd, double ch, double* __restrict__ out, const int* __restrict__ only_unassigned,
           const int* __restrict__ after_founder) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;
  if (g >= P) return;
  // speciation rounds only need genomes still without a species (and, for a
  // founding round, after the founder): skip the rest without touching HBM
  if (only_unassigned && only_unassigned[g] >= 0) return;
  if (after_founder && (after_founder[0] < 0 || g <= after_founder[0])) return;
  double* tile = reinterpret_cast<double*>(smem_raw) + size_t(warp) * S * 33;
  distance_warp(nodes + size_t(g) * N * kNodeCols, conns + size_t(g) * C * kConnCols, rn, S, t, N, C, cd, ch,
                tile, out + size_t(g) * S);
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
  p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  t.n = reinterpret_cast<NSlot*>(p); p += size_t(S) * t.Hn * sizeof(NSlot);
  t.c = reinterpret_cast<CSlot*>(p); p += size_t(S) * t.Hc * sizeof(CSlot);
  t.crow = reinterpret_cast<int*>(p); p += size_t(S) * t.Hc * 4;
  t.counts = reinterpret_cast<int*>(p); p += size_t(S) * 8;
  if (size_t(p - static_cast<uint8_t*>(scratch)) > scratch_bytes) return cudaErrorInvalidValue;
  k_rep_tables<<<S, 256, 0, st>>>(rn, rc, N, C, t);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t per_warp = size_t(S) * 33 * sizeof(double);
  int warps = 4;
  while (warps > 1 && per_warp * warps > 96 * 1024) warps >>= 1;
  const size_t smem = per_warp * warps;
  e = cudaFuncSetAttribute(k_distance, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  k_distance<<<(P + warps - 1) / warps, 32 * warps, smem, st>>>(nodes, conns, P, rn, rc, S, t, N, C, cd, ch, out,
                                                                only_unassigned, after_founder);
  return cudaGetLastError();
}

size_t distance_scratch_bytes(int S, int N, int C) { return rep_tables_bytes(S, N, C); }

}  // namespace fnb
