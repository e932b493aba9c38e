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
  double* cw;                 // [S][Hc] weight of the slot's (lowest) row: a hit needs no row load
  int* counts;                // [S][2] non-empty node / conn rows
  int Hn, Hc;
  // connection-key Bloom filters (one hash bit per key), [S][1 << fw_log2]
  // words; k_distance reads a shared-memory copy.  null = no filter.
  const uint32_t* filt;
  int fw_log2;
};

// filter bit of a key: the hash's high bits (the tables probe from the low
// bits), so a miss in the filter is a miss in the table
__device__ __forceinline__ uint32_t filter_bit(unsigned long long key, int fw_log2) {
  return hash_key(key) >> (32 - (fw_log2 + 5));
}
__device__ __forceinline__ bool filter_has(const uint32_t* f, uint32_t b) { return (f[b >> 5] >> (b & 31)) & 1u; }

constexpr int kLookupBatch = 8;  // representatives whose first probes are issued together

// slot of `key` in a table whose first probe (at `pos`) already returned k0
__device__ __forceinline__ int probe_from(const unsigned long long* keys, int mask, uint32_t pos,
                                          unsigned long long k0, unsigned long long key) {
  while (k0 != key && k0 != kEmptyKey) {
    pos = (pos + 1) & uint32_t(mask);
    k0 = keys[pos];
  }
  return k0 == key ? int(pos) : -1;
}

// Marker tables of one representative (n, c) by the whole CTA.  Ends with
// __syncthreads(); `counts` receives the non-empty node / conn row counts.
__device__ inline void rep_table_build(const double* __restrict__ n, const double* __restrict__ c, int N, int C,
                                       unsigned long long* nk, int* nr, int Hn, unsigned long long* ck, int* cr,
                                       double* cw, int Hc, int* counts) {
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
  for (int i = threadIdx.x; i < Hc; i += blockDim.x) cw[i] = ck[i] != kEmptyKey ? c[cr[i] * kConnCols + kW] : 0.0;
  if (threadIdx.x < 2) counts[threadIdx.x] = cnt[threadIdx.x];
  __syncthreads();
}

// One warp: distance(genome (gn, gc), rep s) for s < S (<= 32); lane s
// writes out[s].  `tile` is this warp's S * 33 doubles of shared memory.
// Rows go in chunks of 32, one row per lane (coalesced genome reads): each
// lane looks its row's marker up in every representative's table and writes
// the row's term for rep s -- node (|db| + |dr| + [agg!=] + [act!=]) / 4,
// connection |dw| / 1, separately rounded (__dadd_rn & co, no contraction),
// +0.0 when unmatched -- into tile[s][row]; then lane s adds the chunk's 32
// terms in row order.  Adding +0.0 for an unmatched row is exact (every term
// is >= +0 and the sums start at +0), so each sum is the reference's g1
// row-order sum bit for bit (ops.hpp:428-441, 454-463).  The argument order
// distance(genome, representative) is kept: 7% of random pairs are bitwise
// asymmetric.
__device__ inline void distance_warp(const double* __restrict__ gn, const double* __restrict__ gc,
                                     const double* __restrict__ rn, const double* __restrict__ rc, int S,
                                     const RepTables& t, int N, int C, double cd, double ch, double* tile,
                                     double* out) {
  const int lane = threadIdx.x & 31;
  int n1 = 0, c1 = 0, mn = 0, mc = 0;
  double sum_n = 0.0, sum_c = 0.0;
  for (int r0 = 0; r0 < N; r0 += 32) {
    const int r = r0 + lane;
    const double* a = gn + size_t(r) * kNodeCols;
    const double k = r < N ? a[kKey] : __longlong_as_double(0x7ff8000000000000ll);
    const bool ne = !isnan(k);
    n1 += __popc(__ballot_sync(0xffffffffu, ne));
    const unsigned long long key = ne ? node_key(k) : 0ull;
    const uint32_t h = hash_key(key) & uint32_t(t.Hn - 1);
    for (int s0 = 0; s0 < S; s0 += kLookupBatch) {
      unsigned long long k0[kLookupBatch];
#pragma unroll
      for (int i = 0; i < kLookupBatch; ++i)  // first probes of several reps in flight
        k0[i] = (ne && s0 + i < S) ? t.nkeys[uint32_t(s0 + i) * uint32_t(t.Hn) + h] : kEmptyKey;
#pragma unroll
      for (int i = 0; i < kLookupBatch; ++i) {
        const int s = s0 + i;
        if (s >= S) break;  // warp-uniform
        const int slot = ne ? probe_from(t.nkeys + size_t(s) * t.Hn, t.Hn - 1, h, k0[i], key) : -1;
        const int q = slot >= 0 ? t.nrows[size_t(s) * t.Hn + slot] : -1;
        double v = 0.0;
        if (q >= 0) {
          const double* b = rn + size_t(s) * N * kNodeCols + size_t(q) * kNodeCols;
          double d = __dadd_rn(fabs(__dsub_rn(a[kBias], b[kBias])), fabs(__dsub_rn(a[kResp], b[kResp])));
          d = __dadd_rn(d, a[kAgg] != b[kAgg] ? 1.0 : 0.0);
          d = __dadd_rn(d, a[kAct] != b[kAct] ? 1.0 : 0.0);
          v = __dmul_rn(d, 0.25);  // == d / 4.0 exactly (both correctly rounded d/4)
        }
        const int m = __popc(__ballot_sync(0xffffffffu, q >= 0));
        if (lane == s) mn += m;
        tile[s * 33 + lane] = v;
      }
    }
    __syncwarp();
    if (lane < S) {
      const int n = min(32, N - r0);
      for (int i = 0; i < n; ++i) sum_n = __dadd_rn(sum_n, tile[lane * 33 + i]);
    }
    __syncwarp();
  }
  for (int r0 = 0; r0 < C; r0 += 32) {
    const int r = r0 + lane;
    double in = __longlong_as_double(0x7ff8000000000000ll), o = 0.0, w = 0.0;
    if (r < C) {
      const double2 x = *reinterpret_cast<const double2*>(gc + size_t(r) * kConnCols);
      in = x.x;
      o = x.y;
    }
    const bool ne = !isnan(in);
    if (ne) w = gc[size_t(r) * kConnCols + kW];
    c1 += __popc(__ballot_sync(0xffffffffu, ne));
    const unsigned long long key = ne ? conn_key(in, o) : 0ull;
    const uint32_t fb = filter_bit(key, t.fw_log2);
    const uint32_t h = hash_key(key) & uint32_t(t.Hc - 1);
    for (int s0 = 0; s0 < S; s0 += kLookupBatch) {
      unsigned long long k0[kLookupBatch];
      uint32_t maybe = 0u;
#pragma unroll
      for (int i = 0; i < kLookupBatch; ++i) {  // filter tests, then first probes in flight
        const int s = s0 + i;
        const bool m = ne && s < S && (!t.filt || filter_has(t.filt + (size_t(s) << t.fw_log2), fb));
        maybe |= uint32_t(m) << i;
        k0[i] = m ? t.ckeys[uint32_t(s) * uint32_t(t.Hc) + h] : kEmptyKey;
      }
#pragma unroll
      for (int i = 0; i < kLookupBatch; ++i) {
        const int s = s0 + i;
        if (s >= S) break;  // warp-uniform
        const int slot = ((maybe >> i) & 1u) ? probe_from(t.ckeys + size_t(s) * t.Hc, t.Hc - 1, h, k0[i], key) : -1;
        // |dw| / 1.0 == |dw| exactly (IEEE division by one)
        const double v = slot >= 0 ? fabs(__dsub_rn(w, t.cw[uint32_t(s) * uint32_t(t.Hc) + uint32_t(slot)])) : 0.0;
        const int m = __popc(__ballot_sync(0xffffffffu, slot >= 0));
        if (lane == s) mc += m;
        tile[s * 33 + lane] = v;
      }
    }
    __syncwarp();
    if (lane < S) {
      const int n = min(32, C - r0);
      for (int i = 0; i < n; ++i) sum_c = __dadd_rn(sum_c, tile[lane * 33 + i]);
    }
    __syncwarp();
  }
  if (lane < S) {
    const int s = lane;
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
