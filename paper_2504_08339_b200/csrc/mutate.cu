// mutate.cu -- K6 (mutate, ops.hpp:196-374) and K7 (InnovationTable
// first-occurrence key handout in slot order, ops.hpp:145-175), bit-exact.
//
// Population mutation in the reference is the sequence
//   plan_node_split (parallel) -> InnovationTable (serial, slot order)
//   -> apply_node_split + mutate_rest (parallel)       (ops.hpp:169-175)
// and the GPU keeps exactly that phase split:
//   k_mutate_plan   one warp per child: stream split(0) decides the split;
//   k7_* kernels    pair -> lowest planning slot (hash + atomicMin), a
//                   slot-order scan of first occurrences, key = next_key+rank;
//   k_mutate_apply  one warp per child: split(1) new node + two connections,
//                   split(2) connection add (16 probes, then the sorted
//                   fallback scan, with creates_cycle answered from a
//                   reachability closure bitset), split(3) node delete,
//                   split(4) connection delete, split(5) attribute pass.
// Row scans (first empty row, k-th enabled row, cascades) are warp ballots;
// every RngStream is owned by lane 0 so its draws are consumed in exactly
// the reference order.  The attribute pass walks the split(5) stream on
// lane 0 recording where each normal() starts, then all lanes evaluate the
// glibc-exact normals (glibc_math.cuh) and apply them.
#include <climits>

#include "fnb_common.cuh"
#include "glibc_math.cuh"
#include "keytable.cuh"
#include "philox.cuh"

namespace fnb {

constexpr unsigned kFullMask = 0xffffffffu;

struct MutCfgDev {
  double node_add, node_delete, conn_add, conn_delete;
  double b_mean, b_std, b_power, b_rate, b_replace;
  double r_mean, r_std, r_power, r_rate, r_replace;
  double w_mean, w_std, w_power, w_rate, w_replace;
  double act_rate, agg_rate;
  int n_act, n_agg, default_act, default_agg;
};

__device__ __forceinline__ Key4 load_key(const uint32_t* keys, int c) {
  return Key4{{keys[4 * c], keys[4 * c + 1], keys[4 * c + 2], keys[4 * c + 3]}};
}

__device__ __forceinline__ bool row_empty_n(const double* n, int r) { return isnan(n[r * kNodeCols + kKey]); }
__device__ __forceinline__ bool row_empty_c(const double* c, int r) { return isnan(c[r * kConnCols + kIn]); }

// lowest row index in [0, n) with pred(row), or -1 (warp-uniform)
template <class F>
__device__ __forceinline__ int warp_first(int n, F pred) {
  const int lane = threadIdx.x & 31;
  for (int r0 = 0; r0 < n; r0 += 32) {
    const unsigned b = __ballot_sync(kFullMask, r0 + lane < n && pred(r0 + lane));
    if (b) return r0 + __ffs(b) - 1;
  }
  return -1;
}
template <class F>
__device__ __forceinline__ int warp_count(int n, F pred) {
  const int lane = threadIdx.x & 31;
  int c = 0;
  for (int r0 = 0; r0 < n; r0 += 32) c += __popc(__ballot_sync(kFullMask, r0 + lane < n && pred(r0 + lane)));
  return c;
}
// row of the k-th (0-based, row order) row with pred(row), or -1
template <class F>
__device__ __forceinline__ int warp_kth(int n, int k, F pred) {
  const int lane = threadIdx.x & 31;
  for (int r0 = 0; r0 < n; r0 += 32) {
    unsigned b = __ballot_sync(kFullMask, r0 + lane < n && pred(r0 + lane));
    const int c = __popc(b);
    if (k < c) {
      for (int i = 0; i < k; ++i) b &= b - 1;
      return r0 + __ffs(b) - 1;
    }
    k -= c;
  }
  return -1;
}

// ---------------------------------------------------------------------------
// plan_node_split (ops.hpp:196-217)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128)
k_mutate_plan(const double* __restrict__ nodes, const double* __restrict__ conns, const uint32_t* __restrict__ keys,
              int n_children, const uint8_t* __restrict__ active, int N, int C, MutCfgDev cfg,
              unsigned long long* __restrict__ plan_pair, int* __restrict__ plan_flag) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= n_children) return;
  int split = 0;
  unsigned long long pair = 0;
  if ((!active || active[c]) && cfg.node_add > 0.0) {
    const double* n = nodes + size_t(c) * N * kNodeCols;
    const double* cc = conns + size_t(c) * C * kConnCols;
    Stream s(key_split(load_key(keys, c), 0));
    int coin = 0;
    if (lane == 0) coin = s.coin(cfg.node_add);
    coin = __shfl_sync(kFullMask, coin, 0);
    if (coin) {
      auto enabled = [&](int r) { return !row_empty_c(cc, r) && cc[r * kConnCols + kEn] == 1.0; };
      const int n_en = warp_count(C, enabled);
      const bool has_node_row = warp_first(N, [&](int r) { return row_empty_n(n, r); }) >= 0;
      const int free_rows = warp_count(C, [&](int r) { return row_empty_c(cc, r); });
      if (n_en > 0 && has_node_row && free_rows >= 2) {
        int idx = 0;
        if (lane == 0) idx = s.index(n_en);
        idx = __shfl_sync(kFullMask, idx, 0);
        const int pick = warp_kth(C, idx, enabled);
        split = 1;
        pair = conn_key(cc[pick * kConnCols + kIn], cc[pick * kConnCols + kOut]);
      }
    }
  }
  if (lane == 0) {
    plan_flag[c] = split;
    plan_pair[c] = pair;
  }
}

// ---------------------------------------------------------------------------
// K7: innovation keys -- first occurrence in slot order wins (ops.hpp:149-156)
// ---------------------------------------------------------------------------
__global__ void k7_init(unsigned long long* tkeys, int* tmin, int H) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < H) { tkeys[i] = kEmptyKey; tmin[i] = INT_MAX; }
}
__global__ void k7_insert(const unsigned long long* __restrict__ pair, const int* __restrict__ flag, int n,
                          unsigned long long* tkeys, int* tmin, int H) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n && flag[c]) table_insert(tkeys, tmin, H - 1, pair[c], c);
}
// single-CTA scan of first-occurrence flags in slot order -> rank[c]
__global__ void __launch_bounds__(1024)
k7_rank(const unsigned long long* __restrict__ pair, const int* __restrict__ flag, int n,
        const unsigned long long* tkeys, const int* tmin, int H, int* __restrict__ rank, int* __restrict__ next_key) {
  __shared__ int warp_sums[32];
  const int t = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int lo = min(n, t * per), hi = min(n, lo + per);
  int cnt = 0;
  for (int c = lo; c < hi; ++c)
    if (flag[c] && table_find(tkeys, tmin, H - 1, pair[c]) == c) ++cnt;
  // block exclusive scan of cnt
  const int lane = t & 31, w = t >> 5;
  int incl = cnt;
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(kFullMask, incl, d);
    if (lane >= d) incl += v;
  }
  if (lane == 31) warp_sums[w] = incl;
  __syncthreads();
  if (w == 0) {
    int v = lane < (nt >> 5) ? warp_sums[lane] : 0;
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(kFullMask, v, d);
      if (lane >= d) v += u;
    }
    warp_sums[lane] = v;  // inclusive
  }
  __syncthreads();
  int base = (w > 0 ? warp_sums[w - 1] : 0) + incl - cnt;
  for (int c = lo; c < hi; ++c) {
    rank[c] = -1;
    if (flag[c] && table_find(tkeys, tmin, H - 1, pair[c]) == c) rank[c] = base++;
  }
  if (t == nt - 1) next_key[1] = warp_sums[(nt >> 5) - 1];  // distinct new pairs
}
__global__ void k7_assign(const unsigned long long* __restrict__ pair, const int* __restrict__ flag, int n,
                          const unsigned long long* tkeys, const int* tmin, int H, const int* __restrict__ rank,
                          const int* __restrict__ next_key, int* __restrict__ new_key) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  new_key[c] = flag[c] ? next_key[0] + rank[table_find(tkeys, tmin, H - 1, pair[c])] : -1;
}
__global__ void k7_advance(int* next_key) { next_key[0] += next_key[1]; }

// ---------------------------------------------------------------------------
// apply_node_split + mutate_rest (ops.hpp:222-361)
// ---------------------------------------------------------------------------
struct MutSmem {
  unsigned long long* nkeys;  // node key -> first row
  int* nrows;
  unsigned long long* ckeys;  // conn pair -> first row
  int* crows;
  uint32_t* reach;            // [N][W]: rows reachable (>= 1 enabled edge) from row
  uint32_t* act_n;            // [2N] bias / response actions of node rows
  uint32_t* act_c;            // [C] weight actions
};

__host__ __device__ inline size_t mut_smem_bytes(int N, int C) {
  const int W = (N + 31) / 32;
  return size_t(table_capacity(N)) * 12 + size_t(table_capacity(C)) * 12 + size_t(N) * W * 4 +
         size_t(2 * N + C) * 4 + 64;
}

__device__ inline MutSmem mut_carve(uint8_t* p, int N, int C) {
  MutSmem s;
  const int Hn = table_capacity(N), Hc = table_capacity(C), W = (N + 31) / 32;
  s.nkeys = reinterpret_cast<unsigned long long*>(p); p += size_t(Hn) * 8;
  s.ckeys = reinterpret_cast<unsigned long long*>(p); p += size_t(Hc) * 8;
  s.nrows = reinterpret_cast<int*>(p); p += size_t(Hn) * 4;
  s.crows = reinterpret_cast<int*>(p); p += size_t(Hc) * 4;
  s.reach = reinterpret_cast<uint32_t*>(p); p += size_t(N) * W * 4;
  s.act_n = reinterpret_cast<uint32_t*>(p); p += size_t(2 * N) * 4;
  s.act_c = reinterpret_cast<uint32_t*>(p);
  return s;
}

__device__ __forceinline__ bool is_key_in(int key, const int* ks, int n) {
  for (int i = 0; i < n; ++i)
    if (ks[i] == key) return true;
  return false;
}

// attribute action code: bit0-1 kind (0 none, 1 add normal(0,power), 2 replace
// normal(init)), bits 2.. = stream position of the normal's first draw
__device__ __forceinline__ uint32_t scalar_action(Stream& s, double rate, double replace) {
  const double u = s.uniform();  // mutate_scalar, ops.hpp:281-289
  if (u < rate || u < rate + replace) {
    const uint32_t pos = uint32_t(s.position());
    s.next_u64();
    s.next_u64();
    return (pos << 2) | (u < rate ? 1u : 2u);
  }
  return 0u;
}

__device__ __forceinline__ double apply_scalar(double v, uint32_t a, const Key4& k, double power, double mean,
                                               double sd) {
  if ((a & 3u) == 0) return v;
  const uint64_t pos = a >> 2;
  const double u0 = u64_to_uniform(stream_u64_at(k, pos)), u1 = u64_to_uniform(stream_u64_at(k, pos + 1));
  if ((a & 3u) == 1) return __dadd_rn(v, glibc::normal_from_uniforms(u0, u1, 0.0, power));
  return glibc::normal_from_uniforms(u0, u1, mean, sd);
}

__global__ void __launch_bounds__(128)
k_mutate_apply(double* __restrict__ nodes, double* __restrict__ conns, const uint32_t* __restrict__ keys,
               int n_children, const uint8_t* __restrict__ active, int N, int C, MutCfgDev cfg, DevShape sh,
               const int* __restrict__ plan_flag, const unsigned long long* __restrict__ plan_pair,
               const int* __restrict__ new_key, int* __restrict__ status, size_t smem_per_warp) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= n_children) return;
  if (active && !active[c]) {
    if (lane == 0) status[c] = 0;
    return;
  }
  MutSmem sm = mut_carve(smem_raw + size_t(warp) * smem_per_warp, N, C);
  double* n = nodes + size_t(c) * N * kNodeCols;
  double* cc = conns + size_t(c) * C * kConnCols;
  const Key4 key = load_key(keys, c);
  const int Hn = table_capacity(N), Hc = table_capacity(C), W = (N + 31) / 32;
  int st = 0;
  auto node_key_at = [&](int r) { return int(n[r * kNodeCols + kKey]); };

  // ---- apply_node_split (ops.hpp:222-243)
  if (plan_flag[c]) {
    const unsigned long long pr = plan_pair[c];
    const int in_key = int(uint32_t(pr >> 32)), out_key = int(uint32_t(pr));
    const int r = warp_first(C, [&](int q) {
      return !row_empty_c(cc, q) && int(cc[q * kConnCols + kIn]) == in_key && int(cc[q * kConnCols + kOut]) == out_key;
    });
    if (r >= 0) {
      const double old_w = cc[r * kConnCols + kW];
      const int nk = new_key[c];
      double bias = 0.0, resp = 0.0;
      if (lane == 0) {
        cc[r * kConnCols + kEn] = 0.0;
        Stream s(key_split(key, 1));
        const double a0 = s.uniform(), a1 = s.uniform(), b0 = s.uniform(), b1 = s.uniform();
        bias = glibc::normal_from_uniforms(a0, a1, cfg.b_mean, cfg.b_std);
        resp = glibc::normal_from_uniforms(b0, b1, cfg.r_mean, cfg.r_std);
      }
      __syncwarp();
      // add_node (ops.hpp:19-27): duplicate key, then first empty row
      const bool dup = warp_first(N, [&](int q) { return !row_empty_n(n, q) && node_key_at(q) == nk; }) >= 0;
      const int nr = warp_first(N, [&](int q) { return row_empty_n(n, q); });
      if (dup) st = 1 + FNB_E_DUPLICATE_KEY;
      else if (nr < 0) st = 1 + FNB_E_GENOME_FULL;
      if (!st) {
        if (lane == 0) {
          double* row = n + nr * kNodeCols;
          row[kKey] = double(nk);
          row[kBias] = bias;
          row[kResp] = resp;
          row[kAgg] = double(cfg.default_agg);
          row[kAct] = double(cfg.default_act);
        }
        __syncwarp();
        // add_conn x2 (ops.hpp:46-58): endpoints exist, pairs are new, first empty row
        for (int e = 0; e < 2 && !st; ++e) {
          const int cr = warp_first(C, [&](int q) { return row_empty_c(cc, q); });
          if (cr < 0) { st = 1 + FNB_E_GENOME_FULL; break; }
          if (lane == 0) {
            double* row = cc + cr * kConnCols;
            row[kIn] = double(e == 0 ? in_key : nk);
            row[kOut] = double(e == 0 ? nk : out_key);
            row[kEn] = 1.0;
            row[kW] = e == 0 ? 1.0 : old_w;
          }
          __syncwarp();
        }
      }
    }
  }

  // ---- connection add (ops.hpp:300-310, pick_new_conn 251-279)
  if (!st && cfg.conn_add > 0.0) {
    Stream s(key_split(key, 2));
    int coin = 0;
    if (lane == 0) coin = s.coin(cfg.conn_add);
    coin = __shfl_sync(kFullMask, coin, 0);
    const int free_row = coin ? warp_first(C, [&](int q) { return row_empty_c(cc, q); }) : -1;
    if (free_row >= 0) {
      auto is_target = [&](int q) { return !row_empty_n(n, q) && !is_key_in(node_key_at(q), sh.input_keys, sh.I); };
      const int nk = warp_count(N, [&](int q) { return !row_empty_n(n, q); });
      const int nt = warp_count(N, is_target);
      if (nk > 0 && nt > 0) {
        // marker tables and the enabled-edge reachability closure (by row)
        for (int i = lane; i < Hn; i += 32) { sm.nkeys[i] = kEmptyKey; sm.nrows[i] = INT_MAX; }
        for (int i = lane; i < Hc; i += 32) { sm.ckeys[i] = kEmptyKey; sm.crows[i] = INT_MAX; }
        for (int i = lane; i < N * W; i += 32) sm.reach[i] = 0u;
        __syncwarp();
        for (int q = lane; q < N; q += 32)
          if (!row_empty_n(n, q)) table_insert(sm.nkeys, sm.nrows, Hn - 1, node_key(n[q * kNodeCols]), q);
        for (int q = lane; q < C; q += 32)
          if (!row_empty_c(cc, q))
            table_insert(sm.ckeys, sm.crows, Hc - 1, conn_key(cc[q * kConnCols + kIn], cc[q * kConnCols + kOut]), q);
        __syncwarp();
        for (int q = lane; q < C; q += 32) {
          if (row_empty_c(cc, q) || cc[q * kConnCols + kEn] != 1.0) continue;
          const int a = table_find(sm.nkeys, sm.nrows, Hn - 1, node_key(cc[q * kConnCols + kIn]));
          const int b = table_find(sm.nkeys, sm.nrows, Hn - 1, node_key(cc[q * kConnCols + kOut]));
          if (a >= 0 && b >= 0) atomicOr(&sm.reach[a * W + (b >> 5)], 1u << (b & 31));
        }
        __syncwarp();
        for (int k = 0; k < N; ++k) {  // Warshall on bitsets
          for (int i = lane; i < N; i += 32)
            if ((sm.reach[i * W + (k >> 5)] >> (k & 31)) & 1u)
              for (int w = 0; w < W; ++w) sm.reach[i * W + w] |= sm.reach[k * W + w];
          __syncwarp();
        }
        // legal(from, to): pair absent and !creates_cycle (ops.hpp:93-111, 261-263)
        auto legal = [&](int from, int to) {
          if (table_find(sm.ckeys, sm.crows, Hc - 1, conn_key(double(from), double(to))) >= 0) return false;
          if (from == to) return false;
          const int rt = table_find(sm.nkeys, sm.nrows, Hn - 1, node_key(double(to)));
          const int rf = table_find(sm.nkeys, sm.nrows, Hn - 1, node_key(double(from)));
          if (rt < 0 || rf < 0) return true;
          return !((sm.reach[rt * W + (rf >> 5)] >> (rf & 31)) & 1u);
        };
        int found = 0, pf = 0, pt = 0;
        if (lane == 0) {
          for (int probe = 0; probe < 16 && !found; ++probe) {
            const int ki = s.index(nk), ti = s.index(nt);
            // keys[] / targets[] are node keys in row order
            int from = 0, to = 0;
            for (int q = 0, seen = 0; q < N; ++q)
              if (!row_empty_n(n, q) && seen++ == ki) { from = node_key_at(q); break; }
            for (int q = 0, seen = 0; q < N; ++q)
              if (!row_empty_n(n, q) && !is_key_in(node_key_at(q), sh.input_keys, sh.I) && seen++ == ti) {
                to = node_key_at(q);
                break;
              }
            if (legal(from, to)) { found = 1; pf = from; pt = to; }
          }
        }
        found = __shfl_sync(kFullMask, found, 0);
        if (!found) {
          // deterministic fallback: sorted keys x sorted targets, from-major
          // (ops.hpp:271-278).  Sorted position of a row = rank of its key.
          int* sk = reinterpret_cast<int*>(sm.act_c);  // scratch: sorted keys / targets
          int* stg = sk + N;
          for (int q = lane; q < N; q += 32) {
            if (row_empty_n(n, q)) continue;
            const int kq = node_key_at(q);
            int rk = 0, rt = 0;
            for (int p = 0; p < N; ++p) {
              if (row_empty_n(n, p)) continue;
              const int kp = node_key_at(p);
              const bool before = kp < kq || (kp == kq && p < q);
              rk += before;
              if (!is_key_in(kp, sh.input_keys, sh.I)) rt += before;
            }
            sk[rk] = kq;
            if (!is_key_in(kq, sh.input_keys, sh.I)) stg[rt] = kq;
          }
          __syncwarp();
          // count legal candidates per `from` (lane-strided), prefix in order
          int total = 0;
          for (int f0 = 0; f0 < nk; f0 += 32) {
            const int f = f0 + lane;
            int cnt = 0;
            if (f < nk)
              for (int t = 0; t < nt; ++t) cnt += legal(sk[f], stg[t]);
            int incl = cnt;
            for (int d = 1; d < 32; d <<= 1) {
              const int v = __shfl_up_sync(kFullMask, incl, d);
              if (lane >= d) incl += v;
            }
            total += __shfl_sync(kFullMask, incl, 31);
          }
          if (total > 0) {
            int idx = 0;
            if (lane == 0) idx = s.index(total);
            idx = __shfl_sync(kFullMask, idx, 0);
            if (lane == 0) {
              for (int f = 0; f < nk && !found; ++f)
                for (int t = 0; t < nt; ++t)
                  if (legal(sk[f], stg[t]) && idx-- == 0) { found = 1; pf = sk[f]; pt = stg[t]; break; }
            }
            found = __shfl_sync(kFullMask, found, 0);
          }
          __syncwarp();
        }
        if (found) {
          pf = __shfl_sync(kFullMask, pf, 0);
          pt = __shfl_sync(kFullMask, pt, 0);
          if (lane == 0) {
            const double u0 = s.uniform(), u1 = s.uniform();
            double* row = cc + free_row * kConnCols;
            row[kIn] = double(pf);
            row[kOut] = double(pt);
            row[kEn] = 1.0;
            row[kW] = glibc::normal_from_uniforms(u0, u1, cfg.w_mean, cfg.w_std);
          }
          __syncwarp();
        }
      }
    }
  }

  // ---- node delete (ops.hpp:311-324)
  if (!st && cfg.node_delete > 0.0) {
    Stream s(key_split(key, 3));
    int coin = 0;
    if (lane == 0) coin = s.coin(cfg.node_delete);
    coin = __shfl_sync(kFullMask, coin, 0);
    if (coin) {
      auto hidden = [&](int q) {
        if (row_empty_n(n, q)) return false;
        const int k = node_key_at(q);
        return !is_key_in(k, sh.input_keys, sh.I) && !is_key_in(k, sh.output_keys, sh.O);
      };
      const int nh = warp_count(N, hidden);
      if (nh > 0) {
        int idx = 0;
        if (lane == 0) idx = s.index(nh);
        idx = __shfl_sync(kFullMask, idx, 0);
        const int rr = warp_kth(N, idx, hidden);
        const int dk = node_key_at(rr);
        // remove_node (ops.hpp:30-44): first row with the key, then cascade
        const int rm = warp_first(N, [&](int q) { return !row_empty_n(n, q) && node_key_at(q) == dk; });
        __syncwarp();
        if (lane == 0)
          for (int a = 0; a < kNodeCols; ++a) n[rm * kNodeCols + a] = __longlong_as_double(0x7ff8000000000000ll);
        for (int q = lane; q < C; q += 32) {
          if (row_empty_c(cc, q)) continue;
          if (int(cc[q * kConnCols + kIn]) == dk || int(cc[q * kConnCols + kOut]) == dk)
            for (int a = 0; a < kConnCols; ++a) cc[q * kConnCols + a] = __longlong_as_double(0x7ff8000000000000ll);
        }
        __syncwarp();
      }
    }
  }

  // ---- connection delete (ops.hpp:325-337)
  if (!st && cfg.conn_delete > 0.0) {
    Stream s(key_split(key, 4));
    int coin = 0;
    if (lane == 0) coin = s.coin(cfg.conn_delete);
    coin = __shfl_sync(kFullMask, coin, 0);
    if (coin) {
      auto live = [&](int q) { return !row_empty_c(cc, q); };
      const int nr = warp_count(C, live);
      if (nr > 0) {
        int idx = 0;
        if (lane == 0) idx = s.index(nr);
        idx = __shfl_sync(kFullMask, idx, 0);
        const int rr = warp_kth(C, idx, live);
        const int a = int(cc[rr * kConnCols + kIn]), b = int(cc[rr * kConnCols + kOut]);
        const int rm = warp_first(C, [&](int q) {
          return !row_empty_c(cc, q) && int(cc[q * kConnCols + kIn]) == a && int(cc[q * kConnCols + kOut]) == b;
        });
        __syncwarp();
        if (lane == 0)
          for (int k = 0; k < kConnCols; ++k) cc[rm * kConnCols + k] = __longlong_as_double(0x7ff8000000000000ll);
        __syncwarp();
      }
    }
  }

  // ---- attributes (ops.hpp:338-359): lane 0 walks split(5), all lanes apply
  if (!st) {
    const Key4 k5 = key_split(key, 5);
    if (lane == 0) {
      Stream s(k5);
      for (int q = 0; q < N; ++q) {
        sm.act_n[2 * q] = 0u;
        sm.act_n[2 * q + 1] = 0u;
        if (row_empty_n(n, q)) continue;
        if (is_key_in(node_key_at(q), sh.input_keys, sh.I)) continue;
        sm.act_n[2 * q] = scalar_action(s, cfg.b_rate, cfg.b_replace);
        sm.act_n[2 * q + 1] = scalar_action(s, cfg.r_rate, cfg.r_replace);
        if (cfg.agg_rate > 0.0 && s.coin(cfg.agg_rate)) n[q * kNodeCols + kAgg] = double(s.index(cfg.n_agg));
        if (cfg.act_rate > 0.0 && s.coin(cfg.act_rate)) n[q * kNodeCols + kAct] = double(s.index(cfg.n_act));
      }
      for (int q = 0; q < C; ++q)
        sm.act_c[q] = row_empty_c(cc, q) ? 0u : scalar_action(s, cfg.w_rate, cfg.w_replace);
    }
    __syncwarp();
    for (int q = lane; q < N; q += 32) {
      const uint32_t ab = sm.act_n[2 * q], ar = sm.act_n[2 * q + 1];
      if (ab) n[q * kNodeCols + kBias] = apply_scalar(n[q * kNodeCols + kBias], ab, k5, cfg.b_power, cfg.b_mean, cfg.b_std);
      if (ar) n[q * kNodeCols + kResp] = apply_scalar(n[q * kNodeCols + kResp], ar, k5, cfg.r_power, cfg.r_mean, cfg.r_std);
    }
    for (int q = lane; q < C; q += 32) {
      const uint32_t aw = sm.act_c[q];
      if (aw) cc[q * kConnCols + kW] = apply_scalar(cc[q * kConnCols + kW], aw, k5, cfg.w_power, cfg.w_mean, cfg.w_std);
    }
  }
  if (lane == 0) status[c] = st;
}

// ---------------------------------------------------------------------------
// host launcher: plan -> K7 -> apply, all on `st`
// ---------------------------------------------------------------------------
size_t mutate_scratch_bytes(int n) {
  const size_t H = size_t(table_capacity(n));
  return size_t(n) * (8 + 4 + 4 + 4) + H * 12 + 64;
}

cudaError_t launch_mutate(double* nodes, double* conns, const uint32_t* keys, int n, const uint8_t* active,
                          const fnb_mutation_config* m, const DevShape& sh, int* d_next_key, int* d_status,
                          void* scratch, size_t scratch_bytes, int* d_new_key_out, cudaStream_t st,
                          long long* launches) {
  if (n <= 0) return cudaSuccess;
  const int N = sh.N, C = sh.C;
  MutCfgDev cfg{m->node_add, m->node_delete, m->conn_add, m->conn_delete,
                m->bias.init_mean, m->bias.init_std, m->bias.mutate_power, m->bias.mutate_rate, m->bias.replace_rate,
                m->response.init_mean, m->response.init_std, m->response.mutate_power, m->response.mutate_rate,
                m->response.replace_rate,
                m->weight.init_mean, m->weight.init_std, m->weight.mutate_power, m->weight.mutate_rate,
                m->weight.replace_rate,
                m->activation_replace_rate, m->aggregation_replace_rate, sh.n_act, sh.n_agg, sh.default_act,
                sh.default_agg};
  const int H = table_capacity(n);
  uint8_t* p = static_cast<uint8_t*>(scratch);
  auto* pair = reinterpret_cast<unsigned long long*>(p); p += size_t(n) * 8;
  auto* tkeys = reinterpret_cast<unsigned long long*>(p); p += size_t(H) * 8;
  int* flag = reinterpret_cast<int*>(p); p += size_t(n) * 4;
  int* rank = reinterpret_cast<int*>(p); p += size_t(n) * 4;
  int* newk = d_new_key_out ? d_new_key_out : reinterpret_cast<int*>(p);
  p += size_t(n) * 4;
  int* tmin = reinterpret_cast<int*>(p); p += size_t(H) * 4;
  if (size_t(p - static_cast<uint8_t*>(scratch)) > scratch_bytes) return cudaErrorInvalidValue;
  const int wpb = 4;
  k_mutate_plan<<<(n + wpb - 1) / wpb, 32 * wpb, 0, st>>>(nodes, conns, keys, n, active, N, C, cfg, pair, flag);
  k7_init<<<(H + 255) / 256, 256, 0, st>>>(tkeys, tmin, H);
  k7_insert<<<(n + 255) / 256, 256, 0, st>>>(pair, flag, n, tkeys, tmin, H);
  k7_rank<<<1, 1024, 0, st>>>(pair, flag, n, tkeys, tmin, H, rank, d_next_key);
  k7_assign<<<(n + 255) / 256, 256, 0, st>>>(pair, flag, n, tkeys, tmin, H, rank, d_next_key, newk);
  k7_advance<<<1, 1, 0, st>>>(d_next_key);
  const size_t per_warp = align16(mut_smem_bytes(N, C));
  int warps = 4;
  while (warps > 1 && per_warp * warps > 96 * 1024) warps >>= 1;
  cudaError_t e = cudaFuncSetAttribute(k_mutate_apply, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(per_warp * warps));
  if (e != cudaSuccess) return e;
  k_mutate_apply<<<(n + warps - 1) / warps, 32 * warps, per_warp * warps, st>>>(
      nodes, conns, keys, n, active, N, C, cfg, sh, flag, pair, newk, d_status, per_warp);
  *launches += 7;
  return cudaGetLastError();
}

}  // namespace fnb
