// distance.cu -- K3: compatibility distance of every genome against S
// species representatives (distance, ops.hpp:415-473), FP64, bit-exact.
//
// The reference walks g1's rows in row order, looks each marker up in g2 by
// linear scan and accumulates the attribute differences sequentially.  Here:
//   * each representative gets an open-addressing marker table once
//     (k_rep_tables), so every lookup is ~1 probe instead of an O(C) scan;
//   * phase A (all 32 lanes, rows strided): markers of the genome are looked
//     up in all S tables, the matched rows kept in shared memory;
//   * phase B (lane s = representative s): the sequential FP64 sums run in
//     exactly g1 row order with separately rounded ops (__dadd_rn & co, no
//     FMA contraction), so the result equals the reference bit for bit
//     (7% of random pairs are bitwise asymmetric -- SURVEY.md H4 -- so the
//     argument order distance(genome, representative) is kept).
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

__host__ inline size_t rep_tables_bytes(int S, int N, int C) {
  const size_t hn = size_t(table_capacity(N)), hc = size_t(table_capacity(C));
  return size_t(S) * (hn * 12 + hc * 12 + 8) + 64;
}

__global__ void k_rep_tables(const double* __restrict__ rn, const double* __restrict__ rc, int N, int C,
                             RepTables t) {
  const int s = blockIdx.x;
  unsigned long long* nk = t.nkeys + size_t(s) * t.Hn;
  int* nr = t.nrows + size_t(s) * t.Hn;
  unsigned long long* ck = t.ckeys + size_t(s) * t.Hc;
  int* cr = t.crows + size_t(s) * t.Hc;
  for (int i = threadIdx.x; i < t.Hn; i += blockDim.x) { nk[i] = kEmptyKey; nr[i] = 0x7fffffff; }
  for (int i = threadIdx.x; i < t.Hc; i += blockDim.x) { ck[i] = kEmptyKey; cr[i] = 0x7fffffff; }
  __shared__ int cnt[2];
  if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
  __syncthreads();
  const double* n = rn + size_t(s) * N * kNodeCols;
  const double* c = rc + size_t(s) * C * kConnCols;
  for (int r = threadIdx.x; r < N; r += blockDim.x) {
    const double k = n[r * kNodeCols + kKey];
    if (isnan(k)) continue;
    table_insert(nk, nr, t.Hn - 1, node_key(k), r);
    atomicAdd(&cnt[0], 1);
  }
  for (int r = threadIdx.x; r < C; r += blockDim.x) {
    const double in = c[r * kConnCols + kIn];
    if (isnan(in)) continue;
    table_insert(ck, cr, t.Hc - 1, conn_key(in, c[r * kConnCols + kOut]), r);
    atomicAdd(&cnt[1], 1);
  }
  __syncthreads();
  if (threadIdx.x < 2) t.counts[2 * s + threadIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(128)
k_distance(const double* __restrict__ nodes, const double* __restrict__ conns, int P,
           const double* __restrict__ rn, const double* __restrict__ rc, int S, RepTables t, int N, int C,
           double cd, double ch, double* __restrict__ out, const int* __restrict__ only_unassigned,
           const int* __restrict__ after_founder) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;
  if (g >= P) return;
  // speciation rounds only need genomes still without a species (and, for a
  // founding round, after the founder): skip the rest without touching HBM
  if (only_unassigned && only_unassigned[g] >= 0) return;
  if (after_founder && (after_founder[0] < 0 || g <= after_founder[0])) return;
  int16_t* match = reinterpret_cast<int16_t*>(smem_raw) + size_t(warp) * S * (N + C);
  const double* gn = nodes + size_t(g) * N * kNodeCols;
  const double* gc = conns + size_t(g) * C * kConnCols;

  // ---- phase A: marker lookups, rows across lanes
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

  // ---- phase B: lane s accumulates rep s in g1 row order (ops.hpp:428-441, 454-463)
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
    out[size_t(g) * S + s] = total;
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
  t.crows = reinterpret_cast<int*>(p); p += size_t(S) * t.Hc * 4;
  t.counts = reinterpret_cast<int*>(p); p += size_t(S) * 8;
  if (size_t(p - static_cast<uint8_t*>(scratch)) > scratch_bytes) return cudaErrorInvalidValue;
  k_rep_tables<<<S, 256, 0, st>>>(rn, rc, N, C, t);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t per_warp = size_t(S) * (N + C) * sizeof(int16_t);
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
