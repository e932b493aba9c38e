// distance_warp.cuh -- the K3 building blocks shared by k_distance
// (distance.cu) and the fused founding rounds (evolve.cu):
//   * rep_table_build: one CTA fills a representative's marker tables
//     (global or shared memory -- the table ops take generic pointers);
//   * distance_warp: one warp computes distance(genome, rep_s) for s < S,
//     bit-exact with distance() (ops.hpp:415-473); lane s writes out[s].
#pragma once
#include "fnb_common.cuh"
#include "keytable.cuh"

namespace fnb {

struct RepTables {
  unsigned long long* nkeys;  // [S][Hn]
  int* nrows;
  unsigned long long* ckeys;  // [S][Hc]
  int* crows;
  int* counts;                // [S][2] non-empty node / conn rows
  int Hn, Hc;
};

// Marker tables of one representative (n, c) by the whole CTA.  Ends with
// __syncthreads(); `counts` receives the non-empty node / conn row counts.
__device__ inline void rep_table_build(const double* __restrict__ n, const double* __restrict__ c, int N, int C,
                                       unsigned long long* nk, int* nr, int Hn, unsigned long long* ck, int* cr,
                                       int Hc, int* counts) {
  __shared__ int cnt[2];
  for (int i = threadIdx.x; i < Hn; i += blockDim.x) { nk[i] = kEmptyKey; nr[i] = 0x7fffffff; }
  for (int i = threadIdx.x; i < Hc; i += blockDim.x) { ck[i] = kEmptyKey; cr[i] = 0x7fffffff; }
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < N; r += blockDim.x) {
    const double k = n[r * kNodeCols + kKey];
    if (isnan(k)) continue;
    table_insert(nk, nr, Hn - 1, node_key(k), r);
    atomicAdd(&cnt[0], 1);
  }
  for (int r = threadIdx.x; r < C; r += blockDim.x) {
    const double in = c[r * kConnCols + kIn];
    if (isnan(in)) continue;
    table_insert(ck, cr, Hc - 1, conn_key(in, c[r * kConnCols + kOut]), r);
    atomicAdd(&cnt[1], 1);
  }
  __syncthreads();
  if (threadIdx.x < 2) counts[threadIdx.x] = cnt[threadIdx.x];
  __syncthreads();
}

// One warp: distance(genome (gn, gc), rep s) for s < S.  `match` is this
// warp's S * (N + C) int16 scratch (shared memory).
//   phase A (all 32 lanes, rows strided): markers looked up in all S tables;
//   phase B (lane s = representative s): the sequential FP64 sums in exactly
//   g1 row order with separately rounded ops (__dadd_rn & co, no FMA
//   contraction), so the result equals the reference bit for bit (7% of
//   random pairs are bitwise asymmetric -- SURVEY.md H4 -- so the argument
//   order distance(genome, representative) is kept).
__device__ inline void distance_warp(const double* __restrict__ gn, const double* __restrict__ gc,
                                     const double* __restrict__ rn, const double* __restrict__ rc, int S,
                                     const RepTables& t, int N, int C, double cd, double ch, int16_t* match,
                                     double* out) {
  const int lane = threadIdx.x & 31;
  int n1 = 0, c1 = 0;
  for (int r0 = 0; r0 < N; r0 += 32) {
    const int r = r0 + lane;
    const double k = r < N ? gn[r * kNodeCols + kKey] : __longlong_as_double(0x7ff8000000000000ll);
    const bool ne = !isnan(k);
    n1 += __popc(__ballot_sync(0xffffffffu, ne));
    if (r < N)
      for (int s = 0; s < S; ++s)
        match[s * (N + C) + r] = int16_t(
            ne ? table_find(t.nkeys + size_t(s) * t.Hn, t.nrows + size_t(s) * t.Hn, t.Hn - 1, node_key(k)) : -1);
  }
  for (int r0 = 0; r0 < C; r0 += 32) {
    const int r = r0 + lane;
    double in = __longlong_as_double(0x7ff8000000000000ll), o = 0.0;
    if (r < C) {
      const double2 a = *reinterpret_cast<const double2*>(gc + r * kConnCols);
      in = a.x;
      o = a.y;
    }
    const bool ne = !isnan(in);
    c1 += __popc(__ballot_sync(0xffffffffu, ne));
    if (r < C) {
      const unsigned long long key = ne ? conn_key(in, o) : 0ull;
      for (int s = 0; s < S; ++s)
        match[s * (N + C) + N + r] =
            int16_t(ne ? table_find(t.ckeys + size_t(s) * t.Hc, t.crows + size_t(s) * t.Hc, t.Hc - 1, key) : -1);
    }
  }
  __syncwarp();

  // phase B: lane s accumulates rep s in g1 row order (ops.hpp:428-441, 454-463)
  for (int s = lane; s < S; s += 32) {
    const int16_t* m = match + s * (N + C);
    const double* rnode = rn + size_t(s) * N * kNodeCols;
    const double* rconn = rc + size_t(s) * C * kConnCols;
    int mn = 0, mc = 0;
    double sum_n = 0.0, sum_c = 0.0;
    for (int r = 0; r < N; ++r) {
      const int q = m[r];
      if (q < 0) continue;
      ++mn;
      const double* a = gn + r * kNodeCols;
      const double* b = rnode + q * kNodeCols;
      double d = __dadd_rn(fabs(__dsub_rn(a[kBias], b[kBias])), fabs(__dsub_rn(a[kResp], b[kResp])));
      d = __dadd_rn(d, a[kAgg] != b[kAgg] ? 1.0 : 0.0);
      d = __dadd_rn(d, a[kAct] != b[kAct] ? 1.0 : 0.0);
      sum_n = __dadd_rn(sum_n, __ddiv_rn(d, 4.0));
    }
    for (int r = 0; r < C; ++r) {
      const int q = m[N + r];
      if (q < 0) continue;
      ++mc;
      sum_c = __dadd_rn(sum_c, __ddiv_rn(fabs(__dsub_rn(gc[r * kConnCols + kW], rconn[q * kConnCols + kW])), 1.0));
    }
    const int n2 = t.counts[2 * s], c2 = t.counts[2 * s + 1];
    double total = 0.0;
    {
      const int disjoint = (n1 - mn) + (n2 - mn);
      const int norm = max(1, max(n1, n2));
      total = __dadd_rn(total, __ddiv_rn(__dmul_rn(cd, double(disjoint)), double(norm)));
      if (mn > 0) total = __dadd_rn(total, __ddiv_rn(__dmul_rn(ch, sum_n), double(mn)));
    }
    {
      const int disjoint = (c1 - mc) + (c2 - mc);
      const int norm = max(1, max(c1, c2));
      total = __dadd_rn(total, __ddiv_rn(__dmul_rn(cd, double(disjoint)), double(norm)));
      if (mc > 0) total = __dadd_rn(total, __ddiv_rn(__dmul_rn(ch, sum_c), double(mc)));
    }
    out[s] = total;
  }
}

}  // namespace fnb
