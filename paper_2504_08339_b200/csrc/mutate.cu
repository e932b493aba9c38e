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
//                   successor bitsets + per-probe BFS; the closure only for
//                   the exhaustive fallback), split(3) node delete,
//                   split(4) connection delete, split(5) attribute pass.
// Row scans (first empty row, k-th enabled row, cascades) are warp ballots;
// every RngStream is owned by lane 0 so its draws are consumed in exactly
// the reference order.  The attribute pass evaluates every decision of the
// split(5) stream per position in parallel (AttrDecider), walks the node
// attributes on lane 0 and the connection weights as a warp-parallel
// automaton (conn_walk), then all lanes evaluate the glibc-exact normals
// (glibc_math.cuh) and apply them.
#include <climits>

#include <cstdlib>

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
k_mutate_plan(const double* __restrict__ nodes, const double* __restrict__ conns, const int32_t* __restrict__ src,
              const uint32_t* __restrict__ keys, int n_children, const uint8_t* __restrict__ active, int N, int C,
              MutCfgDev cfg, unsigned long long* __restrict__ plan_pair, int* __restrict__ plan_flag) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= n_children) return;
  int split = 0;
  unsigned long long pair = 0;
  if ((!active || active[c]) && cfg.node_add > 0.0) {
    // the plan reads only structure (keys, endpoints, enabled flags, empty
    // rows), which a crossover child inherits unchanged from its fit parent
    // (ops.hpp:382-407): `src` lets the plan run on that parent instead
    const size_t gsrc = size_t(src ? src[c] : c);
    const double* n = nodes + gsrc * N * kNodeCols;
    const double* cc = conns + gsrc * C * kConnCols;
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
// first occurrence of each slot's pair (grid-wide; the lookups stay out of the scan)
__global__ void k7_first(const unsigned long long* __restrict__ pair, const int* __restrict__ flag, int n,
                         const unsigned long long* tkeys, const int* tmin, int H, int* __restrict__ rank) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) rank[c] = flag[c] && table_find(tkeys, tmin, H - 1, pair[c]) == c ? 1 : 0;
}
// single-CTA scan of the first-occurrence flags in slot order -> rank[c] (-1: not first)
__global__ void __launch_bounds__(1024)
k7_rank(int n, int* __restrict__ rank, int* __restrict__ next_key) {
  __shared__ int warp_sums[32];
  const int t = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int lo = min(n, t * per), hi = min(n, lo + per);
  int cnt = 0;
  for (int c = lo; c < hi; ++c) cnt += rank[c];
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
  for (int c = lo; c < hi; ++c) rank[c] = rank[c] ? base++ : -1;
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
//
// The child's keys and flags are staged in shared memory (and kept in step
// with every structural edit lane 0 makes to the HBM rows), so each scan
// and each lane-0 stream step is a shared-memory access, not an L2 trip.
// The attribute pass split(5) runs afterwards in its own kernel
// (k_mutate_attrs) with a small footprint.
// ---------------------------------------------------------------------------
struct MutSmem {
  unsigned long long* nkeys;  // marker table: node key -> first row
  int* nrows;
  uint32_t* pairs;             // [N][W]: live connection (from row, to row) present (find_conn, ops.hpp:261)
  uint32_t* reach;            // [N][W]: rows reachable (>= 1 enabled edge) from row
  int* sbuf;                  // [2N] S2 fallback: sorted keys / targets
  int* nkey;                  // [N] node key (rows)
  int* cin;                   // [C]
  int* cout;                  // [C]
  int* list_a;                // [N] scratch lists (keys / targets / sorted)
  int* list_b;                // [N]
  uint8_t* nflag;             // [N] bit0 non-empty, bit1 input, bit2 output
  uint8_t* cflag;             // [C] bit0 non-empty, bit1 enabled
  int* probe;                 // [32] the 16 candidate (from, to) pairs of pick_new_conn
  uint32_t* bfs;              // [3W] visited / frontier / next row bitsets
};

// words of one slot's live-row masks, written by k_mutate_apply from its
// staged flags after the structural edits and read by k_mutate_attrs instead
// of scanning the child's rows again: mutable node rows (non-empty, not an
// input), then live connection rows (non-empty)
__host__ __device__ inline int live_mask_words(int N, int C) { return (N + 31) / 32 + (C + 31) / 32; }

__host__ __device__ inline size_t mut_smem_bytes(int N, int C) {
  const int W = (N + 31) / 32;
  size_t b = size_t(table_capacity(N)) * 12;
  b += size_t(N) * W * 4 * 2 + size_t(2 * N) * 4;  // reach, pairs, sbuf
  b += size_t(N) * 4 * 3 + size_t(C) * 4 * 2;      // nkey, list_a, list_b, cin, cout
  b += size_t(N) + size_t(C) + 64;                 // flags, slack
  b += 32 * 4 + size_t(3 * W) * 4 + 16;            // probes, BFS bitsets
  return align16(b);
}

__device__ inline MutSmem mut_carve(uint8_t* p, int N, int C) {
  MutSmem s;
  const int Hn = table_capacity(N), W = (N + 31) / 32;
  s.nkeys = reinterpret_cast<unsigned long long*>(p); p += size_t(Hn) * 8;
  s.nrows = reinterpret_cast<int*>(p); p += size_t(Hn) * 4;
  s.reach = reinterpret_cast<uint32_t*>(p); p += size_t(N) * W * 4;
  s.pairs = reinterpret_cast<uint32_t*>(p); p += size_t(N) * W * 4;
  s.sbuf = reinterpret_cast<int*>(p); p += size_t(2 * N) * 4;
  s.nkey = reinterpret_cast<int*>(p); p += size_t(N) * 4;
  s.list_a = reinterpret_cast<int*>(p); p += size_t(N) * 4;
  s.list_b = reinterpret_cast<int*>(p); p += size_t(N) * 4;
  s.cin = reinterpret_cast<int*>(p); p += size_t(C) * 4;
  s.cout = reinterpret_cast<int*>(p); p += size_t(C) * 4;
  s.nflag = p; p += N;
  s.cflag = p; p += C;
  p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  s.probe = reinterpret_cast<int*>(p); p += 32 * 4;
  s.bfs = reinterpret_cast<uint32_t*>(p);
  return s;
}

// Warp-collective: is row `dst` reachable from row `src` along the successor
// bitsets succ[N][W] (one enabled edge at least)?  Level-synchronous BFS; it
// touches only the part of the graph below `src`, where the all-pairs closure
// costs N^3/32 bit operations per child.
__device__ inline bool warp_reaches(const uint32_t* succ, int src, int dst, int N, int W, uint32_t* bfs) {
  const int lane = threadIdx.x & 31;
  uint32_t* vis = bfs;
  uint32_t* fr = bfs + W;
  uint32_t* nx = bfs + 2 * W;
  for (int w = lane; w < W; w += 32) {
    const uint32_t b = (src >> 5) == w ? 1u << (src & 31) : 0u;
    vis[w] = 0u;  // src itself counts only if a path returns to it
    fr[w] = b;
    nx[w] = 0u;
  }
  __syncwarp();
  for (;;) {
    for (int q = lane; q < N; q += 32)
      if ((fr[q >> 5] >> (q & 31)) & 1u)
        for (int w = 0; w < W; ++w) {
          const uint32_t v = succ[q * W + w];
          if (v) atomicOr(&nx[w], v);
        }
    __syncwarp();
    bool grew = false;
    for (int w = lane; w < W; w += 32) {
      const uint32_t n = nx[w] & ~vis[w];
      fr[w] = n;
      vis[w] |= n;
      nx[w] = 0u;
      grew = grew || n != 0u;
    }
    __syncwarp();
    if ((vis[dst >> 5] >> (dst & 31)) & 1u) return true;
    if (!__any_sync(kFullMask, grew)) return false;
  }
}

__device__ __forceinline__ bool is_key_in(int key, const int* ks, int n) {
  for (int i = 0; i < n; ++i)
    if (ks[i] == key) return true;
  return false;
}

__device__ __forceinline__ void stage_node(MutSmem& sm, const double* n, int r, const DevShape& sh) {
  const double k = n[r * kNodeCols + kKey];
  if (isnan(k)) { sm.nflag[r] = 0; sm.nkey[r] = 0; return; }
  const int key = int(k);
  sm.nkey[r] = key;
  sm.nflag[r] = uint8_t(1 | (is_key_in(key, sh.input_keys, sh.I) ? 2 : 0) | (is_key_in(key, sh.output_keys, sh.O) ? 4 : 0));
}
__device__ __forceinline__ void stage_conn(MutSmem& sm, const double* c, int r) {
  const double2 a = *reinterpret_cast<const double2*>(c + r * kConnCols);
  if (isnan(a.x)) { sm.cflag[r] = 0; sm.cin[r] = 0; sm.cout[r] = 0; return; }
  sm.cin[r] = int(a.x);
  sm.cout[r] = int(a.y);
  sm.cflag[r] = uint8_t(1 | (c[r * kConnCols + kEn] == 1.0 ? 2 : 0));
}

// attribute action code: bit0-1 kind (0 none, 1 add normal(0,power), 2 replace
// normal(init)), bits 2.. = stream position of the normal's first draw
__device__ __forceinline__ double apply_scalar(double v, uint32_t a, const Key4& k, double power, double mean,
                                               double sd) {
  if ((a & 3u) == 0) return v;
  const uint64_t pos = a >> 2;
  uint32_t b[4];
  stream_block(k, pos >> 1, b);
  uint64_t x0, x1;
  if (pos & 1) {  // draws 2q+1 and 2q+2 straddle two blocks
    x0 = (uint64_t(b[1]) << 32) | b[0];
    stream_block(k, (pos >> 1) + 1, b);
    x1 = (uint64_t(b[3]) << 32) | b[2];
  } else {
    x0 = (uint64_t(b[3]) << 32) | b[2];
    x1 = (uint64_t(b[1]) << 32) | b[0];
  }
  const double u0 = u64_to_uniform(x0), u1 = u64_to_uniform(x1);
  if ((a & 3u) == 1) return __dadd_rn(v, glibc::normal_from_uniforms(u0, u1, 0.0, power));
  return glibc::normal_from_uniforms(u0, u1, mean, sd);
}

// Triggered normals of the attribute pass are not evaluated where the walk
// finds them (a few lanes at a time) but appended to a per-warp list and
// evaluated afterwards with all 32 lanes busy.  Entry: target word
// (bits 30-31 attribute: 0 bias, 1 response, 2 weight; bits 0-29 the double
// offset in the child's node / connection rows) and the action code.
//
// Packed form (one word per entry, when C_max < 2^13 and the window < 2^15):
// bit 31 connection weight, bit 30 replace (else add), bits 15-29 the stream
// position, bits 0-14 the double offset; a node entry's attribute is its
// column (bias / response).  It halves the list, the largest per-warp array.
// (stream positions run past the window only through below() rejections, each
// with probability < 2^-61: the margin to 2^15 is never reached)
__host__ __device__ inline bool normals_packed(int C, int win) { return C < 8192 && win < 30000; }

struct NormalList {
  uint32_t* tgt;
  uint32_t* act;  // unpacked form only
  int* count;
  bool packed;
  __device__ __forceinline__ void put(int i, uint32_t attr, uint32_t off, uint32_t a) const {
    if (packed) {
      tgt[i] = (attr == 2u ? 0x80000000u : 0u) | ((a & 3u) == 2u ? 0x40000000u : 0u) | ((a >> 2) << 15) | off;
    } else {
      tgt[i] = (attr << 30) | off;
      act[i] = a;
    }
  }
  __device__ __forceinline__ void push(uint32_t attr, uint32_t off, uint32_t a) const {
    put(atomicAdd(count, 1), attr, off, a);
  }
  __device__ __forceinline__ void get(int i, uint32_t& attr, uint32_t& off, uint32_t& a) const {
    const uint32_t g = tgt[i];
    if (packed) {
      off = g & 0x7fffu;
      a = (((g >> 15) & 0x7fffu) << 2) | ((g >> 30) & 1u ? 2u : 1u);
      attr = (g >> 31) ? 2u : (off % kNodeCols == kBias ? 0u : 1u);
    } else {
      attr = g >> 30;
      off = g & 0x3fffffffu;
      a = act[i];
    }
  }
};

__device__ __forceinline__ void apply_normals(const NormalList& nl, int total, double* n, double* cc, const Key4& k5,
                                              const MutCfgDev& cfg) {
  for (int t = threadIdx.x & 31; t < total; t += 32) {
    uint32_t attr, off, a;
    nl.get(t, attr, off, a);
    const double power = attr == 0 ? cfg.b_power : attr == 1 ? cfg.r_power : cfg.w_power;
    const double mean = attr == 0 ? cfg.b_mean : attr == 1 ? cfg.r_mean : cfg.w_mean;
    const double sd = attr == 0 ? cfg.b_std : attr == 1 ? cfg.r_std : cfg.w_std;
    double* v = (attr == 2 ? cc : n) + off;
    *v = apply_scalar(*v, a, k5, power, mean, sd);
  }
}

// Every decision the split(5) attribute walk can take at one stream position,
// from that position's draw x (u = uniform(x)):
//   bits 0-1  bias:   u < rate, u < rate + replace   (mutate_scalar, ops.hpp:281-289)
//   bits 2-3  resp:   same
//   bits 4-5  weight: same
//   bit 6/7   u < aggregation / activation replace rate (the coins)
//   bit 8/9   x accepted by below(n_agg) / below(n_act) (rng.hpp:99-106)
//   bits 10-12 / 13-15  x % n_agg / x % n_act (registries hold <= 8)
struct AttrDecider {
  static constexpr int kBias = 0, kResp = 2, kWeight = 4, kAggCoin = 6, kActCoin = 7, kAggAcc = 8, kActAcc = 9,
                       kAggVal = 10, kActVal = 13;
  double b_rate, b_sum, r_rate, r_sum, w_rate, w_sum, agg_rate, act_rate;
  uint64_t lim_agg, lim_act, n_agg, n_act;
  __device__ explicit AttrDecider(const MutCfgDev& c)
      : b_rate(c.b_rate), b_sum(c.b_rate + c.b_replace), r_rate(c.r_rate), r_sum(c.r_rate + c.r_replace),
        w_rate(c.w_rate), w_sum(c.w_rate + c.w_replace), agg_rate(c.agg_rate), act_rate(c.act_rate),
        n_agg(uint64_t(max(1, c.n_agg))), n_act(uint64_t(max(1, c.n_act))) {
    const uint64_t mx = ~0ull;
    lim_agg = mx - ((mx % n_agg) + 1) % n_agg;
    lim_act = mx - ((mx % n_act) + 1) % n_act;
  }
  __device__ __forceinline__ uint16_t operator()(uint64_t x) const {
    const double u = u64_to_uniform(x);
    uint32_t f = uint32_t(u < b_rate) | uint32_t(u < b_sum) << 1 | uint32_t(u < r_rate) << 2 |
                 uint32_t(u < r_sum) << 3 | uint32_t(u < w_rate) << 4 | uint32_t(u < w_sum) << 5 |
                 uint32_t(u < agg_rate) << 6 | uint32_t(u < act_rate) << 7 | uint32_t(x <= lim_agg) << 8 |
                 uint32_t(x <= lim_act) << 9;
    if (agg_rate > 0.0) f |= mod_small(x, uint32_t(n_agg)) << 10;
    if (act_rate > 0.0) f |= mod_small(x, uint32_t(n_act)) << 13;
    return uint16_t(f);
  }
  // x % n for n <= 8 with 32-bit remainders: x = hi * 2^32 + lo
  __device__ __forceinline__ static uint32_t mod_small(uint64_t x, uint32_t n) {
    const uint32_t hi = uint32_t(x >> 32), lo = uint32_t(x);
    const uint32_t r32 = (0u - n) % n;  // 2^32 mod n
    return ((hi % n) * r32 + lo % n) % n;
  }
};

// decision word of a position past the window (only below() rejections get
// there); out of line so the hot chase compiles to a plain branch
__device__ __noinline__ uint32_t slow_word(const Key4& k5, uint32_t q, const AttrDecider& dec) {
  return dec(stream_u64_at(k5, q));
}

// The connection-weight part of the split(5) walk in parallel.  Each live
// connection is one mutate_scalar: at its position p it consumes p and, when
// the weight bits of word p trigger, the two draws of a normal.  As an
// automaton over positions the state is "draws still to skip" (0, 1, 2), so:
// every lane folds its chunk of [p0, p0 + 3m) into a 3-entry state map, a warp
// scan of map compositions gives each chunk's incoming state, a scan of visit
// counts gives each visit's connection index k, and the lane that finds
// visit k lists its normal for the k-th live row.  Returns false (nothing
// listed) when the walk could leave the decision window.
__device__ __forceinline__ uint32_t map_at(uint32_t m, uint32_t s) { return (m >> (2 * s)) & 3u; }

template <typename DW>
__device__ bool conn_walk(const DW* dw, uint32_t need, uint32_t p0, int m, const int16_t* live_row,
                          const NormalList& nl) {
  const int lane = threadIdx.x & 31;
  const uint32_t span = 3u * uint32_t(m);
  if (p0 + span > need) return false;
  const uint32_t L = (span + 31) / 32;
  const uint32_t lo = min(p0 + span, p0 + uint32_t(lane) * L), hi = min(p0 + span, lo + L);
  auto bits = [&](uint32_t p) { return (uint32_t(dw[p]) >> AttrDecider::kWeight) & 3u; };
  // pass 1: this chunk's map of start state -> end state
  uint32_t s0 = 0, s1 = 1, s2 = 2;
  for (uint32_t p = lo; p < hi; ++p) {
    const uint32_t t = bits(p) ? 2u : 0u;
    s0 = s0 ? s0 - 1 : t;
    s1 = s1 ? s1 - 1 : t;
    s2 = s2 ? s2 - 1 : t;
  }
  uint32_t f = s0 | (s1 << 2) | (s2 << 4);
  for (int d = 1; d < 32; d <<= 1) {  // inclusive scan: F_l = f_l o F_{l-1}
    const uint32_t g = __shfl_up_sync(kFullMask, f, d);
    if (lane >= d) f = map_at(f, map_at(g, 0)) | (map_at(f, map_at(g, 1)) << 2) | (map_at(f, map_at(g, 2)) << 4);
  }
  const uint32_t prev = __shfl_up_sync(kFullMask, f, 1);
  const uint32_t s_in = lane == 0 ? 0u : map_at(prev, 0);
  // pass 2: visits in this chunk, exclusive prefix -> first connection index
  uint32_t s = s_in;
  int cnt = 0;
  for (uint32_t p = lo; p < hi; ++p) {
    if (s == 0) {
      ++cnt;
      s = bits(p) ? 2u : 0u;
    } else {
      --s;
    }
  }
  int incl = cnt;
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(kFullMask, incl, d);
    if (lane >= d) incl += v;
  }
  // pass 3: list the triggered normals of this chunk's visits
  int k = incl - cnt;
  s = s_in;
  for (uint32_t p = lo; p < hi; ++p) {
    if (s == 0) {
      const uint32_t b = bits(p);
      if (b && k < m) nl.push(2u, uint32_t(live_row[k]) * kConnCols + kW, ((p + 1) << 2) | ((b & 1u) ? 1u : 2u));
      ++k;
      s = b ? 2u : 0u;
    } else {
      --s;
    }
  }
  return true;
}

// MINB = 8: 8 CTAs (32 warps) per SM where shared memory allows it (C2): the
// kernel is latency-bound (lane-0 streams, warp scans), so occupancy is worth
// a few spilled registers.  MINB = 4 where shared memory holds residency to
// <= 16 warps anyway (C5: 19 KB per warp): registers without spills.
template <int MINB>
__global__ void __launch_bounds__(128, MINB)
k_mutate_apply(double* __restrict__ nodes, double* __restrict__ conns, const uint32_t* __restrict__ keys,
               int n_children, const uint8_t* __restrict__ active, int N, int C, MutCfgDev cfg, DevShape sh,
               const int* __restrict__ plan_flag, const unsigned long long* __restrict__ plan_pair,
               const int* __restrict__ new_key, int* __restrict__ status, size_t smem_per_warp, int l2_prefetch,
               uint32_t* __restrict__ live_mask) {
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
  // the staging loops walk the child chunk by chunk: its rows go to L2 first
  if (l2_prefetch && lane == 0) {
    prefetch_l2_range(cc, size_t(C) * kConnCols * 8);
    prefetch_l2_range(n, size_t(N) * kNodeCols * 8);
  }
  const Key4 key = load_key(keys, c);
  const int Hn = table_capacity(N), W = (N + 31) / 32;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  int st = 0;
  for (int r = lane; r < N; r += 32) stage_node(sm, n, r, sh);
  for (int r = lane; r < C; r += 32) stage_conn(sm, cc, r);
  __syncwarp();
  auto n_live = [&](int q) { return (sm.nflag[q] & 1) != 0; };
  auto c_live = [&](int q) { return (sm.cflag[q] & 1) != 0; };

  // ---- apply_node_split (ops.hpp:222-243)
  if (plan_flag[c]) {
    const unsigned long long pr = plan_pair[c];
    const int in_key = int(uint32_t(pr >> 32)), out_key = int(uint32_t(pr));
    const int r = warp_first(C, [&](int q) { return c_live(q) && sm.cin[q] == in_key && sm.cout[q] == out_key; });
    if (r >= 0) {
      const int nk = new_key[c];
      const bool dup = warp_first(N, [&](int q) { return n_live(q) && sm.nkey[q] == nk; }) >= 0;
      const int nr = warp_first(N, [&](int q) { return !n_live(q); });
      const int cr0 = warp_first(C, [&](int q) { return !c_live(q); });
      const int cr1 = cr0 < 0 ? -1 : warp_first(C, [&](int q) { return q > cr0 && !c_live(q); });
      if (lane == 0) {
        const double old_w = cc[r * kConnCols + kW];
        cc[r * kConnCols + kEn] = 0.0;
        sm.cflag[r] = 1;
        if (dup) st = 1 + FNB_E_DUPLICATE_KEY;          // add_node (ops.hpp:19-27)
        else if (nr < 0) st = 1 + FNB_E_GENOME_FULL;
        else if (cr1 < 0) st = 1 + FNB_E_GENOME_FULL;   // add_conn x2 (ops.hpp:46-58)
        if (!st) {
          Stream s(key_split(key, 1));
          const double a0 = s.uniform(), a1 = s.uniform(), b0 = s.uniform(), b1 = s.uniform();
          double* row = n + nr * kNodeCols;
          row[kKey] = double(nk);
          row[kBias] = glibc::normal_from_uniforms(a0, a1, cfg.b_mean, cfg.b_std);
          row[kResp] = glibc::normal_from_uniforms(b0, b1, cfg.r_mean, cfg.r_std);
          row[kAgg] = double(cfg.default_agg);
          row[kAct] = double(cfg.default_act);
          double* c0 = cc + cr0 * kConnCols;
          c0[kIn] = double(in_key); c0[kOut] = double(nk); c0[kEn] = 1.0; c0[kW] = 1.0;
          double* c1 = cc + cr1 * kConnCols;
          c1[kIn] = double(nk); c1[kOut] = double(out_key); c1[kEn] = 1.0; c1[kW] = old_w;
          sm.nkey[nr] = nk;
          sm.nflag[nr] = uint8_t(1 | (is_key_in(nk, sh.input_keys, sh.I) ? 2 : 0) | (is_key_in(nk, sh.output_keys, sh.O) ? 4 : 0));
          sm.cin[cr0] = in_key; sm.cout[cr0] = nk; sm.cflag[cr0] = 3;
          sm.cin[cr1] = nk; sm.cout[cr1] = out_key; sm.cflag[cr1] = 3;
        }
      }
      st = __shfl_sync(kFullMask, st, 0);
      __syncwarp();
    }
  }

  // ---- connection add (ops.hpp:300-310, pick_new_conn 251-279)
  if (!st && cfg.conn_add > 0.0) {
    Stream s(key_split(key, 2));
    int coin = 0;
    if (lane == 0) coin = s.coin(cfg.conn_add);
    coin = __shfl_sync(kFullMask, coin, 0);
    const int free_row = coin ? warp_first(C, [&](int q) { return !c_live(q); }) : -1;
    if (free_row >= 0) {
      // keys[] (node keys, row order) and targets[] (non-input keys, row order)
      int nk = 0, nt = 0;
      for (int r0 = 0; r0 < N; r0 += 32) {
        const int q = r0 + lane;
        const bool live = q < N && n_live(q);
        const bool tgt = live && !(sm.nflag[q] & 2);
        const unsigned bl = __ballot_sync(kFullMask, live), bt = __ballot_sync(kFullMask, tgt);
        const unsigned below = (1u << lane) - 1u;
        if (live) sm.list_a[nk + __popc(bl & below)] = sm.nkey[q];
        if (tgt) sm.list_b[nt + __popc(bt & below)] = sm.nkey[q];
        nk += __popc(bl);
        nt += __popc(bt);
      }
      if (nk > 0 && nt > 0) {
        for (int i = lane; i < Hn; i += 32) { sm.nkeys[i] = kEmptyKey; sm.nrows[i] = INT_MAX; }
        for (int i = lane; i < N * W; i += 32) { sm.reach[i] = 0u; sm.pairs[i] = 0u; }
        __syncwarp();
        for (int q = lane; q < N; q += 32)
          if (n_live(q)) table_insert(sm.nkeys, sm.nrows, Hn - 1, uint32_t(sm.nkey[q]), q);
        __syncwarp();
        // present pairs over live rows (find_conn) and successor bitsets over
        // enabled edges (ops.hpp:106), both by node row (a key's first row).
        // Probe endpoints are node keys, so a pair whose endpoint has no node
        // row can never match a probe.
        for (int q = lane; q < C; q += 32) {
          if (!c_live(q)) continue;
          const int a = table_find(sm.nkeys, sm.nrows, Hn - 1, uint32_t(sm.cin[q]));
          const int b = table_find(sm.nkeys, sm.nrows, Hn - 1, uint32_t(sm.cout[q]));
          if (a >= 0 && b >= 0) {
            atomicOr(&sm.pairs[a * W + (b >> 5)], 1u << (b & 31));
            if (sm.cflag[q] == 3) atomicOr(&sm.reach[a * W + (b >> 5)], 1u << (b & 31));
          }
        }
        // the 16 probes of pick_new_conn (ops.hpp:256-266): their draws do not
        // depend on the legality of earlier probes, so lane 0 draws them all
        if (lane == 0) {
          const uint64_t lim_k = Stream::below_limit(uint64_t(nk)), lim_t = Stream::below_limit(uint64_t(nt));
          for (int p = 0; p < 16; ++p) {
            sm.probe[2 * p] = sm.list_a[s.index_lim(nk, lim_k)];
            sm.probe[2 * p + 1] = sm.list_b[s.index_lim(nt, lim_t)];
          }
        }
        __syncwarp();
        // sm.reach holds successor bitsets; the fallback below closes it in place
        // legal(from, to): pair absent and !creates_cycle (ops.hpp:93-111, 261-263)
        auto present = [&](int rf, int rt) {  // find_conn(from, to) >= 0
          return rf >= 0 && rt >= 0 && ((sm.pairs[rf * W + (rt >> 5)] >> (rt & 31)) & 1u);
        };
        auto legal = [&](int from, int to) {
          const int rt = table_find(sm.nkeys, sm.nrows, Hn - 1, uint32_t(to));
          const int rf = table_find(sm.nkeys, sm.nrows, Hn - 1, uint32_t(from));
          if (present(rf, rt)) return false;
          if (from == to) return false;
          if (rt < 0 || rf < 0) return true;
          return !((sm.reach[rt * W + (rf >> 5)] >> (rf & 31)) & 1u);
        };
        int found = 0, pf = 0, pt = 0, pidx = -1;
        for (int p = 0; p < 16 && !found; ++p) {  // warp-uniform
          const int from = sm.probe[2 * p], to = sm.probe[2 * p + 1];
          const int rt = table_find(sm.nkeys, sm.nrows, Hn - 1, uint32_t(to));
          const int rf = table_find(sm.nkeys, sm.nrows, Hn - 1, uint32_t(from));
          bool ok = false;
          if (!present(rf, rt) && from != to)
            ok = rt < 0 || rf < 0 || !warp_reaches(sm.reach, rt, rf, N, W, sm.bfs);
          if (ok) {
            found = 1;
            pf = from;
            pt = to;
            pidx = p;
          }
        }
        if (found && lane == 0) {  // the stream right after the accepted probe
          s = Stream(key_split(key, 2));
          s.coin(cfg.conn_add);
          const uint64_t lim_k = Stream::below_limit(uint64_t(nk)), lim_t = Stream::below_limit(uint64_t(nt));
          for (int p = 0; p <= pidx; ++p) {
            s.index_lim(nk, lim_k);
            s.index_lim(nt, lim_t);
          }
        }
        if (!found) {  // all-pairs closure for the fallback enumeration (Warshall on bitsets)
          for (int k = 0; k < N; ++k) {
            for (int i = lane; i < N; i += 32)
              if ((sm.reach[i * W + (k >> 5)] >> (k & 31)) & 1u)
                for (int w = 0; w < W; ++w) sm.reach[i * W + w] |= sm.reach[k * W + w];
            __syncwarp();
          }
        }
        if (!found) {
          // deterministic fallback: sorted keys x sorted targets, from-major
          // (ops.hpp:271-278); sorted position = rank of (key, list index)
          int* sk = sm.sbuf;
          int* stg = sk + N;
          __syncwarp();
          for (int q = lane; q < nk; q += 32) {
            const int kq = sm.list_a[q];
            int rk = 0;
            for (int p = 0; p < nk; ++p) rk += sm.list_a[p] < kq || (sm.list_a[p] == kq && p < q);
            sk[rk] = kq;
          }
          for (int q = lane; q < nt; q += 32) {
            const int kq = sm.list_b[q];
            int rt = 0;
            for (int p = 0; p < nt; ++p) rt += sm.list_b[p] < kq || (sm.list_b[p] == kq && p < q);
            stg[rt] = kq;
          }
          __syncwarp();
          int total = 0;
          for (int f0 = 0; f0 < nk; f0 += 32) {
            const int f = f0 + lane;
            int cnt = 0;
            if (f < nk)
              for (int t = 0; t < nt; ++t) cnt += legal(sk[f], stg[t]);
            for (int d = 16; d > 0; d >>= 1) cnt += __shfl_down_sync(kFullMask, cnt, d);
            total += __shfl_sync(kFullMask, cnt, 0);
          }
          if (total > 0) {
            int idx = 0;
            if (lane == 0) {
              idx = s.index(total);
              for (int f = 0; f < nk && !found; ++f)
                for (int t = 0; t < nt; ++t)
                  if (legal(sk[f], stg[t]) && idx-- == 0) { found = 1; pf = sk[f]; pt = stg[t]; break; }
            }
            found = __shfl_sync(kFullMask, found, 0);
          }
          __syncwarp();
        }
        if (found && lane == 0) {
          const double u0 = s.uniform(), u1 = s.uniform();
          double* row = cc + free_row * kConnCols;
          row[kIn] = double(pf);
          row[kOut] = double(pt);
          row[kEn] = 1.0;
          row[kW] = glibc::normal_from_uniforms(u0, u1, cfg.w_mean, cfg.w_std);
          sm.cin[free_row] = pf;
          sm.cout[free_row] = pt;
          sm.cflag[free_row] = 3;
        }
        __syncwarp();
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
      auto hidden = [&](int q) { return sm.nflag[q] == 1; };  // non-empty, neither input nor output
      const int nh = warp_count(N, hidden);
      if (nh > 0) {
        int idx = 0;
        if (lane == 0) idx = s.index(nh);
        idx = __shfl_sync(kFullMask, idx, 0);
        const int dk = sm.nkey[warp_kth(N, idx, hidden)];
        // remove_node (ops.hpp:30-44): first row with the key, then cascade
        const int rm = warp_first(N, [&](int q) { return n_live(q) && sm.nkey[q] == dk; });
        __syncwarp();
        if (lane == 0) {
          for (int a = 0; a < kNodeCols; ++a) n[rm * kNodeCols + a] = nan;
          sm.nflag[rm] = 0;
        }
        for (int q = lane; q < C; q += 32) {
          if (!c_live(q) || (sm.cin[q] != dk && sm.cout[q] != dk)) continue;
          for (int a = 0; a < kConnCols; ++a) cc[q * kConnCols + a] = nan;
          sm.cflag[q] = 0;
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
      const int nr = warp_count(C, c_live);
      if (nr > 0) {
        int idx = 0;
        if (lane == 0) idx = s.index(nr);
        idx = __shfl_sync(kFullMask, idx, 0);
        const int rr = warp_kth(C, idx, c_live);
        const int a = sm.cin[rr], b = sm.cout[rr];
        const int rm = warp_first(C, [&](int q) { return c_live(q) && sm.cin[q] == a && sm.cout[q] == b; });
        __syncwarp();
        if (lane == 0) {
          for (int k = 0; k < kConnCols; ++k) cc[rm * kConnCols + k] = nan;
          sm.cflag[rm] = 0;
        }
        __syncwarp();
      }
    }
  }

  // the live-row masks of the structurally final child (k_mutate_attrs):
  // lane l builds word l from 32 staged flags
  {
    const int WN = (N + 31) >> 5, WT = live_mask_words(N, C);
    uint32_t* lm = live_mask + size_t(c) * WT;
    for (int w = lane; w < WT; w += 32) {
      const bool node = w < WN;
      const uint8_t* f = node ? sm.nflag + 32 * w : sm.cflag + 32 * (w - WN);
      const int lim = node ? N - 32 * w : C - 32 * (w - WN);
      uint32_t bits = 0;
      for (int i = 0; i < 32 && i < lim; ++i) {
        const uint32_t x = f[i];
        bits |= uint32_t(node ? (x & 3u) == 1u : (x & 1u) != 0u) << i;
      }
      lm[w] = bits;
    }
  }
  if (lane == 0) status[c] = st;
}

// ---------------------------------------------------------------------------
// attributes (ops.hpp:338-359), one warp per child after the structural pass.
// The split(5) walk is sequential (a scalar consumes 1 or 3 draws depending on
// its own draw), so: all lanes first evaluate every decision the walk could
// take at every stream position of a window that covers the worst case (one
// 16-bit word per position, AttrDecider); lane 0 chases the node attributes
// through the words; the connection weights are walked as a warp-parallel
// automaton (conn_walk) that applies their normals; all lanes finally apply
// the node normals.  Positions past the window (only reachable through
// below() rejections) are evaluated directly from the stream.
// ---------------------------------------------------------------------------
__host__ __device__ inline int attr_per_node(const MutCfgDev& cfg) {
  return 6 + (cfg.agg_rate > 0.0 ? 2 : 0) + (cfg.act_rate > 0.0 ? 2 : 0);
}
__host__ __device__ inline int attr_window(int N, int C, int per_node) { return (per_node * N + 3 * C + 1) & ~1; }
// Decision words are one byte when neither activation nor aggregation is ever
// replaced (bits 6-15 of AttrDecider are then never read).
__host__ __device__ inline bool attr_words_narrow(const MutCfgDev& cfg) {
  return !(cfg.agg_rate > 0.0) && !(cfg.act_rate > 0.0);
}
__host__ __device__ inline size_t attr_smem_bytes(int N, int C, int win, bool narrow) {
  return align16(size_t(win) * (narrow ? 1 : 2)) + align16(size_t(C) * 2) +
         (normals_packed(C, win) ? 1 : 2) * align16(size_t(2 * N + C) * 4) + align16(size_t(2 * N)) +
         align16(size_t(N)) + 16;
}

// <= 64 registers (a 4-byte spill): C2 164 -> 157 us, C5 unchanged at 5.0 ms;
// unbounded (104 registers) C5 takes 5.6 ms
template <typename DW>
__global__ void __launch_bounds__(256, 4)
k_mutate_attrs(double* __restrict__ nodes, double* __restrict__ conns, const uint32_t* __restrict__ keys,
               int n_children, const uint8_t* __restrict__ active, const int* __restrict__ status, int N, int C,
               MutCfgDev cfg, DevShape sh, int win, size_t smem_per_warp, int l2_prefetch,
               const uint32_t* __restrict__ live_mask) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= n_children) return;
  if ((active && !active[c]) || status[c]) return;
  uint8_t* p8 = smem_raw + size_t(warp) * smem_per_warp;
  DW* dw = reinterpret_cast<DW*>(p8); p8 += align16(size_t(win) * sizeof(DW));
  int16_t* live_row = reinterpret_cast<int16_t*>(p8); p8 += align16(size_t(C) * 2);
  NormalList nl;
  nl.packed = normals_packed(C, win);
  nl.tgt = reinterpret_cast<uint32_t*>(p8); p8 += align16(size_t(2 * N + C) * 4);
  nl.act = nullptr;
  if (!nl.packed) {
    nl.act = reinterpret_cast<uint32_t*>(p8);
    p8 += align16(size_t(2 * N + C) * 4);
  }
  int8_t* new_id = reinterpret_cast<int8_t*>(p8); p8 += align16(size_t(2 * N));  // [q] agg, [N + q] act
  uint8_t* hid = p8; p8 += align16(size_t(N));                                    // [N] mutable node row
  nl.count = reinterpret_cast<int*>(p8);
  double* n = nodes + size_t(c) * N * kNodeCols;
  double* cc = conns + size_t(c) * C * kConnCols;
  const Key4 k5 = key_split(load_key(keys, c), 5);
  if (l2_prefetch && lane == 0) {  // the rows are read-modify-written after the decision walk
    prefetch_l2_range(cc, size_t(C) * kConnCols * 8);
    prefetch_l2_range(n, size_t(N) * kNodeCols * 8);
  }

  // rows of the structurally final child: mutable nodes, live connections,
  // from the masks k_mutate_apply left (no pass over the rows themselves)
  int nn = 0, nc = 0;
  const uint32_t* lm = live_mask + size_t(c) * live_mask_words(N, C);
  for (int r0 = 0; r0 < N; r0 += 32) {
    const uint32_t b = lm[r0 >> 5];
    const int r = r0 + lane;
    if (r < N) hid[r] = (b >> lane) & 1u;
    nn += __popc(b);
  }
  for (int r0 = 0; r0 < C; r0 += 32) {
    const uint32_t bl = lm[((N + 31) >> 5) + (r0 >> 5)];
    const int r = r0 + lane;
    if ((bl >> lane) & 1u) live_row[nc + __popc(bl & ((1u << lane) - 1u))] = int16_t(r);
    nc += __popc(bl);
  }
  const int need = min(win, (nn * attr_per_node(cfg) + nc * 3 + 1) & ~1);
  const AttrDecider dec(cfg);
  for (int b = lane; 2 * b < need; b += 32) {
    uint32_t w[4];
    stream_block(k5, uint64_t(b), w);
    dw[2 * b] = DW(dec((uint64_t(w[3]) << 32) | w[2]));
    dw[2 * b + 1] = DW(dec((uint64_t(w[1]) << 32) | w[0]));
  }
  __syncwarp();
  uint32_t p_nodes_end = 0;
  if (lane == 0) {  // node attributes: lane 0 chases the decision words in row order
    uint32_t p = 0;
    auto word = [&](uint32_t q) -> uint32_t { return q < uint32_t(need) ? uint32_t(dw[q]) : slow_word(k5, q, dec); };
    auto scalar = [&](int sh_) -> uint32_t {  // mutate_scalar (ops.hpp:281-289): action code
      const uint32_t f = (word(p++) >> sh_) & 3u;
      if (!f) return 0u;
      const uint32_t a = (p << 2) | ((f & 1u) ? 1u : 2u);
      p += 2;
      return a;
    };
    auto index = [&](int acc_bit, int val_shift) -> int {  // below(n), rng.hpp:99-106
      for (;;) {
        const uint32_t f = word(p++);
        if ((f >> acc_bit) & 1u) return int((f >> val_shift) & 7u);
      }
    };
    int listed = 0;
    for (int q = 0; q < N; ++q) {
      int ag = -1, ac = -1;
      if (hid[q]) {
        const uint32_t ab = scalar(AttrDecider::kBias);
        if (ab) {
          nl.put(listed++, 0u, uint32_t(q * kNodeCols + kBias), ab);
        }
        const uint32_t ar = scalar(AttrDecider::kResp);
        if (ar) {
          nl.put(listed++, 1u, uint32_t(q * kNodeCols + kResp), ar);
        }
        if (cfg.agg_rate > 0.0 && ((word(p++) >> AttrDecider::kAggCoin) & 1u))
          ag = index(AttrDecider::kAggAcc, AttrDecider::kAggVal);
        if (cfg.act_rate > 0.0 && ((word(p++) >> AttrDecider::kActCoin) & 1u))
          ac = index(AttrDecider::kActAcc, AttrDecider::kActVal);
      }
      new_id[q] = int8_t(ag);
      new_id[N + q] = int8_t(ac);
    }
    p_nodes_end = p;
    *nl.count = listed;
  }
  __syncwarp();
  // connection weights from p0 (warp-parallel; lane-0 chase if the window is short)
  const uint32_t p0 = __shfl_sync(kFullMask, p_nodes_end, 0);
  if (!conn_walk(dw, uint32_t(need), p0, nc, live_row, nl) && lane == 0) {
    uint32_t p = p0;
    for (int k = 0; k < nc; ++k) {
      const uint32_t f = ((p < uint32_t(need) ? uint32_t(dw[p]) : slow_word(k5, p, dec)) >> AttrDecider::kWeight) & 3u;
      ++p;
      if (f) {
        nl.push(2u, uint32_t(live_row[k]) * kConnCols + kW, (p << 2) | ((f & 1u) ? 1u : 2u));
        p += 2;
      }
    }
  }
  __syncwarp();
  apply_normals(nl, *nl.count, n, cc, k5, cfg);
  for (int q = lane; q < N; q += 32) {
    if (new_id[q] >= 0) n[q * kNodeCols + kAgg] = double(new_id[q]);
    if (new_id[N + q] >= 0) n[q * kNodeCols + kAct] = double(new_id[N + q]);
  }
}

// ---------------------------------------------------------------------------
// host launcher: plan -> K7 -> apply, all on `st`
// ---------------------------------------------------------------------------
size_t mutate_scratch_bytes(int n, int N, int C) {
  const size_t H = size_t(table_capacity(n));
  return size_t(n) * (8 + 4 + 4 + 4) + H * 12 + 64 + size_t(n) * live_mask_words(N, C) * 4 + 16;
}

static MutCfgDev mut_cfg_dev(const fnb_mutation_config* m, const DevShape& sh) {
  return MutCfgDev{m->node_add, m->node_delete, m->conn_add, m->conn_delete,
                   m->bias.init_mean, m->bias.init_std, m->bias.mutate_power, m->bias.mutate_rate, m->bias.replace_rate,
                   m->response.init_mean, m->response.init_std, m->response.mutate_power, m->response.mutate_rate,
                   m->response.replace_rate,
                   m->weight.init_mean, m->weight.init_std, m->weight.mutate_power, m->weight.mutate_rate,
                   m->weight.replace_rate,
                   m->activation_replace_rate, m->aggregation_replace_rate, sh.n_act, sh.n_agg, sh.default_act,
                   sh.default_agg};
}

struct MutScratch {
  unsigned long long *pair, *tkeys;
  int *flag, *rank, *newk, *tmin;
  uint32_t* mask;  // [n][live_mask_words] live-row masks
  int H;
};
static bool mut_scratch(void* scratch, size_t scratch_bytes, int n, int N, int C, int* d_new_key_out,
                        MutScratch* ms) {
  ms->H = table_capacity(n);
  uint8_t* p = static_cast<uint8_t*>(scratch);
  ms->pair = reinterpret_cast<unsigned long long*>(p); p += size_t(n) * 8;
  ms->tkeys = reinterpret_cast<unsigned long long*>(p); p += size_t(ms->H) * 8;
  ms->flag = reinterpret_cast<int*>(p); p += size_t(n) * 4;
  ms->rank = reinterpret_cast<int*>(p); p += size_t(n) * 4;
  ms->newk = d_new_key_out ? d_new_key_out : reinterpret_cast<int*>(p);
  p += size_t(n) * 4;
  ms->tmin = reinterpret_cast<int*>(p); p += size_t(ms->H) * 4;
  p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  ms->mask = reinterpret_cast<uint32_t*>(p); p += size_t(n) * live_mask_words(N, C) * 4;
  return size_t(p - static_cast<uint8_t*>(scratch)) <= scratch_bytes;
}

// the plan arrays inside the scratch (host-layer replay of a caller's InnovationTable)
void mutate_scratch_views(void* scratch, int n, unsigned long long** pair, int** flag, int** newk) {
  MutScratch ms;
  mut_scratch(scratch, size_t(-1), n, 1, 1, nullptr, &ms);
  *pair = ms.pair;
  *flag = ms.flag;
  *newk = ms.newk;
}

// Phase 1 of mutate for n slots: the node-split plan (stream split(0)) and the
// K7 innovation keys, in slot order over ALL n slots.  `src` (may be null)
// maps slot c to the genome its structure is read from (the fit parent).
cudaError_t launch_mutate_plan(const double* nodes, const double* conns, const int32_t* src, const uint32_t* keys,
                               int n, const uint8_t* active, const fnb_mutation_config* m, const DevShape& sh,
                               int* d_next_key, void* scratch, size_t scratch_bytes, int* d_new_key_out,
                               cudaStream_t st, long long* launches) {
  if (n <= 0) return cudaSuccess;
  const MutCfgDev cfg = mut_cfg_dev(m, sh);
  MutScratch ms;
  if (!mut_scratch(scratch, scratch_bytes, n, sh.N, sh.C, d_new_key_out, &ms)) return cudaErrorInvalidValue;
  const int wpb = 4, H = ms.H;
  k_mutate_plan<<<(n + wpb - 1) / wpb, 32 * wpb, 0, st>>>(nodes, conns, src, keys, n, active, sh.N, sh.C, cfg, ms.pair,
                                                          ms.flag);
  k7_init<<<(H + 255) / 256, 256, 0, st>>>(ms.tkeys, ms.tmin, H);
  k7_insert<<<(n + 255) / 256, 256, 0, st>>>(ms.pair, ms.flag, n, ms.tkeys, ms.tmin, H);
  k7_first<<<(n + 255) / 256, 256, 0, st>>>(ms.pair, ms.flag, n, ms.tkeys, ms.tmin, H, ms.rank);
  k7_rank<<<1, 1024, 0, st>>>(n, ms.rank, d_next_key);
  k7_assign<<<(n + 255) / 256, 256, 0, st>>>(ms.pair, ms.flag, n, ms.tkeys, ms.tmin, H, ms.rank, d_next_key,
                                              ms.newk);
  k7_advance<<<1, 1, 0, st>>>(d_next_key);
  *launches += 7;
  return cudaGetLastError();
}

// Phase 2 for slots [lo, hi) of the n planned ones: structural mutations
// (node split with its K7 key, conn add, node / conn delete) and attributes.
// Slots are independent, so any partition of [0, n) gives the same genomes.
cudaError_t launch_mutate_apply(double* nodes, double* conns, const uint32_t* keys, int n, int lo, int hi,
                                const uint8_t* active, const fnb_mutation_config* m, const DevShape& sh,
                                int* d_status, void* scratch, size_t scratch_bytes, const int* d_new_key,
                                cudaStream_t st, long long* launches) {
  if (hi <= lo) return cudaSuccess;
  const int N = sh.N, C = sh.C, k = hi - lo;
  const MutCfgDev cfg = mut_cfg_dev(m, sh);
  MutScratch ms;
  if (!mut_scratch(scratch, scratch_bytes, n, sh.N, sh.C, const_cast<int*>(d_new_key), &ms)) return cudaErrorInvalidValue;
  double* nd = nodes + size_t(lo) * N * kNodeCols;
  double* cd = conns + size_t(lo) * C * kConnCols;
  const uint32_t* ky = keys + 4 * size_t(lo);
  const uint8_t* ac = active ? active + lo : nullptr;
  const size_t per_warp = align16(mut_smem_bytes(N, C));
  const int warps = warps_per_cta_for_smem(per_warp, 4);
  static int smem_sm = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    return v > 0 ? v : 233472;
  }();
  const int resident = int(smem_sm / (per_warp * warps + 1024)) * warps;
  auto apply_kern = resident <= 16 ? k_mutate_apply<4> : k_mutate_apply<8>;
  cudaError_t e = cudaFuncSetAttribute(apply_kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(per_warp * warps));
  if (e != cudaSuccess) return e;
  static const int l2pf = [] {  // experiment knob
    const char* e = std::getenv("FNB_K6_L2PF");
    return e ? std::atoi(e) : 1;
  }();
  apply_kern<<<(k + warps - 1) / warps, 32 * warps, per_warp * warps, st>>>(
      nd, cd, ky, k, ac, N, C, cfg, sh, ms.flag + lo, ms.pair + lo, ms.newk + lo, d_status + lo, per_warp, l2pf,
      ms.mask + size_t(lo) * live_mask_words(N, C));
  const int win = attr_window(N, C, attr_per_node(cfg));
  const bool narrow = attr_words_narrow(cfg);
  const size_t aw = attr_smem_bytes(N, C, win, narrow);
  const int awarps = warps_per_cta_for_smem(aw, 8);
  auto kern = narrow ? k_mutate_attrs<uint8_t> : k_mutate_attrs<uint16_t>;
  static const int l2pf_attrs = [] {  // experiment knob
    const char* e = std::getenv("FNB_K6A_L2PF");
    return e ? std::atoi(e) : 1;
  }();
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(aw * awarps));
  if (e != cudaSuccess) return e;
  kern<<<(k + awarps - 1) / awarps, 32 * awarps, aw * awarps, st>>>(nd, cd, ky, k, ac, d_status + lo, N, C, cfg, sh,
                                                                    win, aw, l2pf_attrs,
                                                                    ms.mask + size_t(lo) * live_mask_words(N, C));
  *launches += 2;
  return cudaGetLastError();
}

// plan -> K7 -> apply over all n slots, on `st`
cudaError_t launch_mutate(double* nodes, double* conns, const uint32_t* keys, int n, const uint8_t* active,
                          const fnb_mutation_config* m, const DevShape& sh, int* d_next_key, int* d_status,
                          void* scratch, size_t scratch_bytes, int* d_new_key_out, cudaStream_t st,
                          long long* launches) {
  cudaError_t e = launch_mutate_plan(nodes, conns, nullptr, keys, n, active, m, sh, d_next_key, scratch,
                                     scratch_bytes, d_new_key_out, st, launches);
  if (e != cudaSuccess) return e;
  MutScratch ms;
  if (!mut_scratch(scratch, scratch_bytes, n, sh.N, sh.C, d_new_key_out, &ms)) return cudaErrorInvalidValue;
  return launch_mutate_apply(nodes, conns, keys, n, 0, n, active, m, sh, d_status, scratch, scratch_bytes, ms.newk,
                             st, launches);
}

}  // namespace fnb
