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

constexpr int kLookupBatch = 8;  // representatives whose first probes are issued together

// Representative tables: open addressing, power-of-two capacity, hash_key
// (keytable.cuh).  A slot is 16 bytes so one load answers a probe:
//   node slot  {key, lowest row}          (attributes read from the rep row)
//   conn slot  {key, weight of the lowest row holding the pair}
// (the reference's find_* scans return the first matching row,
// genome.hpp:195-210).  A row's probe start is the same in every
// representative's table, so lookups for several representatives are issued
// together.
struct NSlot {
  unsigned long long key;
  int row;
  int pad;
};
struct CSlot {
  unsigned long long key;
  double w;
};
static_assert(sizeof(NSlot) == 16 && sizeof(CSlot) == 16, "16-byte table slots");

struct RepTables {
  NSlot* n;      // [S][Hn]
  CSlot* c;      // [S][Hc]
  int* crow;     // [S][Hc] build scratch: lowest conn row per slot
  int* counts;   // [S][2] non-empty node / conn rows
  int Hn, Hc;
};

__host__ __device__ inline size_t rep_table_bytes_one(int N, int C) {
  return size_t(table_capacity(N)) * sizeof(NSlot) + size_t(table_capacity(C)) * (sizeof(CSlot) + 4) + 16;
}

// Marker tables of one representative (n, c) by the whole CTA (global or
// shared memory).  Ends with __syncthreads().
__device__ inline void rep_table_build(const double* __restrict__ n, const double* __restrict__ c, int N, int C,
                                       NSlot* ns, int Hn, CSlot* cs, int* crow, int Hc, int* counts) {
  __shared__ int cnt[2];
  for (int i = threadIdx.x; i < Hn; i += blockDim.x) ns[i] = NSlot{kEmptyKey, 0x7fffffff, 0};
  for (int i = threadIdx.x; i < Hc; i += blockDim.x) {
    cs[i] = CSlot{kEmptyKey, 0.0};
    crow[i] = 0x7fffffff;
  }
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < N; r += blockDim.x) {
    const double k = n[r * kNodeCols + kKey];
    if (isnan(k)) continue;
    const unsigned long long key = node_key(k);
    uint32_t s = hash_key(key) & uint32_t(Hn - 1);
    for (;;) {
      const unsigned long long prev = atomicCAS(&ns[s].key, kEmptyKey, key);
      if (prev == kEmptyKey || prev == key) {
        atomicMin(&ns[s].row, r);
        break;
      }
      s = (s + 1) & uint32_t(Hn - 1);
    }
    atomicAdd(&cnt[0], 1);
  }
  for (int r = threadIdx.x; r < C; r += blockDim.x) {
    const double in = c[r * kConnCols + kIn];
    if (isnan(in)) continue;
    const unsigned long long key = conn_key(in, c[r * kConnCols + kOut]);
    uint32_t s = hash_key(key) & uint32_t(Hc - 1);
    for (;;) {
      const unsigned long long prev = atomicCAS(&cs[s].key, kEmptyKey, key);
      if (prev == kEmptyKey || prev == key) {
        atomicMin(&crow[s], r);
        break;
      }
      s = (s + 1) & uint32_t(Hc - 1);
    }
    atomicAdd(&cnt[1], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < Hc; i += blockDim.x)
    if (cs[i].key != kEmptyKey) cs[i].w = c[crow[i] * kConnCols + kW];
  if (threadIdx.x < 2) counts[threadIdx.x] = cnt[threadIdx.x];
  __syncthreads();
}

// continue a probe sequence whose first slot `x` (at `pos`) was already loaded
template <class Slot>
__device__ __forceinline__ bool probe_rest(const Slot* tab, uint32_t mask, uint32_t pos, unsigned long long key,
                                           Slot& x) {
  while (x.key != key && x.key != kEmptyKey) {
    pos = (pos + 1) & mask;
    x = tab[pos];
  }
  return x.key == key;
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
                                     const double* __restrict__ rn, int S,
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
      NSlot x[kLookupBatch];
#pragma unroll
      for (int i = 0; i < kLookupBatch; ++i)
        if (ne && s0 + i < S) x[i] = t.n[size_t(s0 + i) * t.Hn + h];
#pragma unroll
      for (int i = 0; i < kLookupBatch; ++i) {
        const int s = s0 + i;
        if (s >= S) break;  // warp-uniform
        int q = -1;
        if (ne && probe_rest(t.n + size_t(s) * t.Hn, uint32_t(t.Hn - 1), h, key, x[i])) q = x[i].row;
        double v = 0.0;
        if (q >= 0) {
          const double* b = rn + size_t(s) * N * kNodeCols + size_t(q) * kNodeCols;
          double d = __dadd_rn(fabs(__dsub_rn(a[kBias], b[kBias])), fabs(__dsub_rn(a[kResp], b[kResp])));
          d = __dadd_rn(d, a[kAgg] != b[kAgg] ? 1.0 : 0.0);
          d = __dadd_rn(d, a[kAct] != b[kAct] ? 1.0 : 0.0);
          v = __ddiv_rn(d, 4.0);
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
    const uint32_t h = hash_key(key) & uint32_t(t.Hc - 1);
    for (int s0 = 0; s0 < S; s0 += kLookupBatch) {
      CSlot x[kLookupBatch];
#pragma unroll
      for (int i = 0; i < kLookupBatch; ++i)
        if (ne && s0 + i < S) x[i] = t.c[size_t(s0 + i) * t.Hc + h];
#pragma unroll
      for (int i = 0; i < kLookupBatch; ++i) {
        const int s = s0 + i;
        if (s >= S) break;  // warp-uniform
        const bool hit = ne && probe_rest(t.c + size_t(s) * t.Hc, uint32_t(t.Hc - 1), h, key, x[i]);
        const double v = hit ? __ddiv_rn(fabs(__dsub_rn(w, x[i].w)), 1.0) : 0.0;
        const int m = __popc(__ballot_sync(0xffffffffu, hit));
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
