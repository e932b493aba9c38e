// transform.cu -- K1: per-genome transform (network.hpp:122-220) on sm_100a.
//
// One warp per genome.  The reference builds a dense max_nodes^2 `expanded`
// tensor, runs Kahn's algorithm with a sorted ready list and keeps per-row
// incoming lists; here the enabled graph lives in a per-warp shared-memory
// predecessor bitset (max_nodes bits per row), the min-(key,row) pop of
// network.hpp:192-214 is a warp __reduce_min over node ranks, and the output
// is the compact op/edge program of fnb_common.cuh.  Semantics kept bit for
// bit: error precedence (act id, agg id per row; inputs; outputs; conn rows;
// cycle), duplicate keys resolving to the lowest row (lower_bound over
// (key,row), network.hpp:57-63), in-degree counting per enabled ROW while
// Kahn decrements per distinct cell (so duplicate enabled pairs and NaN
// weights block their target exactly like the reference), the
// initial-ready `key >= 0` filter (network.hpp:195), and incoming edges in
// ascending source row (network.hpp:184-190).
#include "fnb_common.cuh"

namespace fnb {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned long long kHtEmpty = ~0ull;
constexpr int kLastForever = 0x7fffffff;  // last_use of an output row
constexpr uint8_t kNoRow = 0xff;          // (node rows are < FNB_MAX_NODES_LIMIT = 255)

// Per-warp shared memory.  Arrays that die after a step are reused by a later
// one (noted at the reuse).
struct TfSmem {
  long long* kr;        // [N, padded even] (key << 8 | row) or INT64_MAX for empty rows
  unsigned long long* ht;  // [HT] key -> lowest row (key << 32 | row), open addressing
  int* sorted_key;      // [N] key of rank k
  int* R;               // [N] enabled rows per destination row
  uint32_t* pred;       // [N * W] predecessor rows of each row (row bits)
  uint32_t* predr;      // [N * W] predecessor ranks of each rank (rank bits); slot-chain scratch after Kahn
  uint16_t* row_of_rank;// [N]
  uint16_t* rank;       // [N]
  uint16_t* order;      // [N]
  uint16_t* ebeg;       // [N] record begin of the op writing row r (in ht's space after step 4)
  uint16_t* op_row;     // [N] row of op k (in ht's space after step 4)
  uint16_t* ncode;      // [N] act code | agg code << 8
  float* nbias;         // [N]
  float* nresp;         // [N]
  uint8_t* flags;       // [N] bit0 non-empty, bit1 input
  uint8_t* csrc;        // [C] source row (rows fit a byte: N_max <= 255)
  uint8_t* cdst;        // [C] destination row of an enabled finite edge, else kNoRow
  float* cw;            // [C] FP32 weight of an edge row (W <= 2 only)
  uint32_t ht_mask, ht_shift;
};

__host__ __device__ inline int tf_ht_size(int N) {
  int h = 32;
  while (h < 2 * N) h <<= 1;
  return h;
}

__host__ __device__ inline size_t tf_smem_bytes(int N, int C, int W) {
  size_t b = 0;
  b += align16(size_t(N + 1) * 8);       // kr
  b += align16(size_t(tf_ht_size(N)) * 8);  // ht
  b += align16(size_t(N) * 4) * 2;       // sorted_key, R
  b += align16(size_t(N) * W * 4) * 2;   // pred, predr
  b += align16(size_t(N) * 2) * 4;       // row_of_rank, rank, order, ncode
  b += align16(size_t(N) * 4) * 2;       // nbias, nresp
  b += align16(size_t(N));               // flags
  b += align16(size_t(C)) * 2;           // csrc, cdst
  if (W <= 2) b += align16(size_t(C) * 4);  // cw: FP32 weights staged in step 4 (kStageW)
  return b;
}

__device__ inline TfSmem tf_carve(uint8_t* p, int N, int C, int W) {
  TfSmem s;
  s.kr = reinterpret_cast<long long*>(p); p += align16(size_t(N + 1) * 8);
  const int ht = tf_ht_size(N);
  s.ht = reinterpret_cast<unsigned long long*>(p); p += align16(size_t(ht) * 8);
  s.ht_mask = uint32_t(ht - 1);
  s.ht_shift = uint32_t(32 - __ffs(ht) + 1);
  s.sorted_key = reinterpret_cast<int*>(p); p += align16(size_t(N) * 4);
  s.R = reinterpret_cast<int*>(p); p += align16(size_t(N) * 4);
  s.pred = reinterpret_cast<uint32_t*>(p); p += align16(size_t(N) * W * 4);
  s.predr = reinterpret_cast<uint32_t*>(p); p += align16(size_t(N) * W * 4);
  s.row_of_rank = reinterpret_cast<uint16_t*>(p); p += align16(size_t(N) * 2);
  s.rank = reinterpret_cast<uint16_t*>(p); p += align16(size_t(N) * 2);
  s.order = reinterpret_cast<uint16_t*>(p); p += align16(size_t(N) * 2);
  s.ebeg = reinterpret_cast<uint16_t*>(s.ht);  // ht (>= 16N bytes) is dead after step 4
  s.op_row = s.ebeg + N;
  s.ncode = reinterpret_cast<uint16_t*>(p); p += align16(size_t(N) * 2);
  s.nbias = reinterpret_cast<float*>(p); p += align16(size_t(N) * 4);
  s.nresp = reinterpret_cast<float*>(p); p += align16(size_t(N) * 4);
  s.flags = p; p += align16(size_t(N));
  s.csrc = p; p += align16(size_t(C));
  s.cdst = p;
  p += align16(size_t(C));
  s.cw = W <= 2 ? reinterpret_cast<float*>(p) : nullptr;
  return s;
}

__device__ __forceinline__ uint32_t tf_hash(const TfSmem& s, int key) {
  return (uint32_t(key) * 0x9E3779B1u) >> s.ht_shift;
}

// key -> lowest row holding it: the row of the first (key,row) in sorted order,
// i.e. TransformedNetwork::row_of_key's lower_bound (network.hpp:57-63)
__device__ inline void tf_insert(const TfSmem& s, int key, int row) {
  const unsigned long long v = (static_cast<unsigned long long>(uint32_t(key)) << 32) | uint32_t(row);
  uint32_t h = tf_hash(s, key);
  for (;;) {
    const unsigned long long prev = atomicCAS(&s.ht[h], kHtEmpty, v);
    if (prev == kHtEmpty) return;
    if (uint32_t(prev >> 32) == uint32_t(key)) {
      atomicMin(&s.ht[h], v);
      return;
    }
    h = (h + 1) & s.ht_mask;
  }
}

// row of `key`, or -1
__device__ inline int tf_lookup(const TfSmem& s, int key) {
  uint32_t h = tf_hash(s, key);
  for (;;) {
    const unsigned long long v = s.ht[h];
    if (v == kHtEmpty) return -1;
    if (uint32_t(v >> 32) == uint32_t(key)) return int(uint32_t(v));
    h = (h + 1) & s.ht_mask;
  }
}

__device__ inline void tf_fail(uint8_t* net, int status, int kind, int a, int b,
                               int order_count) {
  NetHeader* h = reinterpret_cast<NetHeader*>(net);
  h->status = status;
  h->err_kind = kind;
  h->err_a = a;
  h->err_b = b;
  h->order_count = int16_t(order_count);
  h->n_ops = 0;
  h->n_edges = 0;
  h->n_rec = 0;
  h->n_slots = -2;  // no value-slot count (K2 also skips the genome by its status)
}

// kPk: the genome comes as packed transfer rows (PackedLayout, `packed` +
// g * pk.bytes) instead of the FP64 rows; every derived value is the same
template <int W, bool kPk>
__global__ void __launch_bounds__(128)
k_transform(const double* __restrict__ nodes, const double* __restrict__ conns, const uint8_t* __restrict__ packed,
            int P, uint8_t* __restrict__ nets, NetLayout L, DevShape sh, size_t smem_per_warp) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;
  if (g >= P) return;
  const int N = sh.N, C = sh.C;
  TfSmem s = tf_carve(smem_raw + size_t(warp) * smem_per_warp, N, C, W);
  const double* nrow = kPk ? nullptr : nodes + size_t(g) * N * kNodeCols;
  const double* crow = kPk ? nullptr : conns + size_t(g) * C * kConnCols;
  const PackedLayout pk(N, C);
  const uint8_t* pg = kPk ? packed + size_t(g) * pk.bytes : nullptr;
  uint8_t* net = nets + size_t(g) * L.bytes;

  // ---- 1. node rows: keys, activation/aggregation ids (network.hpp:139-152);
  //         the op attributes are kept in shared memory for step 6d
  for (int i = lane; i <= int(s.ht_mask); i += 32) s.ht[i] = kHtEmpty;
  if (lane == 0) s.kr[N] = 0x7fffffffffffffffll;  // pad for the paired rank loads
  int populated = 0;
  bool narrow = true;  // every key in [-2^23, 2^23 - 1): (key << 8 | row) fits an int32 below INT32_MAX
  for (int r0 = 0; r0 < N; r0 += 32) {
    const int r = r0 + lane;
    int bad = kErrNone, badid = 0;
    bool ne = false;
    if (r < N) {
      const double* row = kPk ? nullptr : nrow + r * kNodeCols;
      int key = 0;
      double rb = 0.0, rr = 0.0, rg = 0.0, ra = 0.0;
      if constexpr (kPk) {
        ne = pg[pk.nflag + r] & 1u;
        key = reinterpret_cast<const int*>(pg + pk.key)[r];
      } else {  // the whole row in one round trip (its columns share two sectors)
        const double k = row[kKey];
        rb = row[kBias];
        rr = row[kResp];
        rg = row[kAgg];
        ra = row[kAct];
        ne = !isnan(k);
        key = int(k);
      }
      long long kr = 0x7fffffffffffffffll;
      if (ne) {
        kr = (static_cast<long long>(key) << 8) | r;
        narrow = narrow && key >= -(1 << 23) && key < (1 << 23) - 1;  // INT32_MAX stays the empty mark
        const int act = kPk ? int(pg[pk.act + r]) : int(ra);
        const int agg = kPk ? int(pg[pk.agg + r]) : int(rg);
        if (act < 0 || act >= sh.n_act) { bad = kErrActId; badid = act; }
        else if (agg < 0 || agg >= sh.n_agg) { bad = kErrAggId; badid = agg; }
        else {
          s.ncode[r] = uint16_t(sh.act[act] | (sh.agg[agg] << 8));
          if constexpr (kPk) {
            s.nbias[r] = reinterpret_cast<const float*>(pg + pk.bias)[r];
            s.nresp[r] = reinterpret_cast<const float*>(pg + pk.resp)[r];
          } else {
            s.nbias[r] = float(rb);
            s.nresp[r] = float(rr);
          }
        }
      }
      s.kr[r] = kr;
      s.flags[r] = ne ? 1 : 0;
      s.R[r] = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) s.pred[r * W + w] = 0u;
#pragma unroll
      for (int w = 0; w < W; ++w) s.predr[r * W + w] = 0u;
    }
    const unsigned m = __ballot_sync(kFull, bad != kErrNone);
    if (m) {
      const int l = __ffs(m) - 1;
      const int kind = __shfl_sync(kFull, bad, l);
      const int id = __shfl_sync(kFull, badid, l);
      if (lane == 0) tf_fail(net, 1 + FNB_E_UNKNOWN_FUNCTION, kind, id, 0, 0);
      return;
    }
    populated += __popc(__ballot_sync(kFull, ne));
  }
  narrow = __all_sync(kFull, narrow);
  __syncwarp();
  if (narrow) {  // repack in place as int32 (INT32_MAX for empty rows), padded to a multiple of 4
    int* k32 = reinterpret_cast<int*>(s.kr);
    int v[W];
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const int r = lane + 32 * j;
      v[j] = 0x7fffffff;
      if (r < N) {
        const long long x = s.kr[r];
        if (x != 0x7fffffffffffffffll) v[j] = int(x);
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const int r = lane + 32 * j;
      if (r < ((N + 3) & ~3)) k32[r] = v[j];
    }
    __syncwarp();
  }

  // ---- 2. ranks of (key,row): the Kahn priority and the key_to_row sort;
  //         the key -> lowest-row hash table
  for (int r = lane; r < N; r += 32) {
    int rk = 0, key;
    if (narrow) {
      const int mine = reinterpret_cast<const int*>(s.kr)[r];
      if (mine == 0x7fffffff) continue;
      const int4* k4 = reinterpret_cast<const int4*>(s.kr);
      for (int q = 0; q < (N + 3) / 4; ++q) {
        const int4 v = k4[q];
        rk += (v.x < mine ? 1 : 0) + (v.y < mine ? 1 : 0) + (v.z < mine ? 1 : 0) + (v.w < mine ? 1 : 0);
      }
      key = mine >> 8;  // arithmetic shift: (key << 8 | row) >> 8 == key
    } else {
      const long long mine = s.kr[r];
      if (mine == 0x7fffffffffffffffll) continue;
      const longlong2* kr2 = reinterpret_cast<const longlong2*>(s.kr);
      for (int q = 0; q < (N + 1) / 2; ++q) {
        const longlong2 v = kr2[q];
        rk += (v.x < mine ? 1 : 0) + (v.y < mine ? 1 : 0);
      }
      key = int(mine >> 8);
    }
    s.rank[r] = uint16_t(rk);
    s.row_of_rank[rk] = uint16_t(r);
    s.sorted_key[rk] = key;
    tf_insert(s, key, r);
  }
  __syncwarp();

  // ---- 3. inputs then outputs (network.hpp:155-165)
  // lane i keeps input / output i's row in a register (I, O <= 32); the net
  // block receives their value slots in step 8
  uint16_t* in_rows = reinterpret_cast<uint16_t*>(net + L.in_off);
  uint16_t* out_rows = reinterpret_cast<uint16_t*>(net + L.out_off);
  int my_in = -1, my_out = -1;
  for (int pass = 0; pass < 2; ++pass) {
    const int n = pass == 0 ? sh.I : sh.O;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      int row = 0, key = 0;
      if (i < n) {
        key = pass == 0 ? sh.input_keys[i] : sh.output_keys[i];
        row = tf_lookup(s, key);
      }
      const unsigned m = __ballot_sync(kFull, i < n && row < 0);
      if (m) {
        const int l = __ffs(m) - 1;
        const int k = __shfl_sync(kFull, key, l);
        if (lane == 0)
          tf_fail(net, 1 + FNB_E_DANGLING_ENDPOINT, pass == 0 ? kErrInputKey : kErrOutputKey, k, 0, 0);
        return;
      }
      if (i < n) {
        if (pass == 0) { my_in = row; s.flags[row] |= 2; }
        else my_out = row;
      }
    }
  }
  __syncwarp();

  // ---- 4. connection rows: dangling check, in-degree, predecessor bits in
  //         row and rank space (network.hpp:167-183)
  const uint64_t keep = l2_keep();  // the weights are read again in step 7
  // rows of the next two 32-row chunks are in flight while a chunk is processed
  // (FP64 rows: {in, out} and {enabled, w}; packed: in, out, w bits, flags)
  const double2 kNoConn = make_double2(__longlong_as_double(0x7ff8000000000000ll), 0.0);
  double2 qa0 = kNoConn, qb0 = kNoConn, qa1 = kNoConn, qb1 = kNoConn;
  auto load_conn = [&](int r, double2& a, double2& b) {
    if constexpr (kPk) {  // the packed fields ride in the double2 registers
      const int in = reinterpret_cast<const int*>(pg + pk.cin)[r];
      const int out = reinterpret_cast<const int*>(pg + pk.cout)[r];
      const float w = reinterpret_cast<const float*>(pg + pk.w)[r];
      const uint32_t f = pg[pk.cflag + r];
      a = make_double2(__hiloint2double(int(f), in), 0.0);
      b = make_double2(__hiloint2double(out, __float_as_int(w)), 0.0);
    } else {
      a = ld2_l2(crow + r * kConnCols, keep);
      b = ld2_l2(crow + r * kConnCols + 2, keep);
    }
  };
  if (lane < C) load_conn(lane, qa0, qb0);
  if (32 + lane < C) load_conn(32 + lane, qa1, qb1);
  for (int r0 = 0; r0 < C; r0 += 32) {
    const int r = r0 + lane;
    const double2 a = qa0, b = qb0;
    qa0 = qa1;
    qb0 = qb1;
    qa1 = kNoConn;
    qb1 = kNoConn;
    if (r + 64 < C) load_conn(r + 64, qa1, qb1);
    bool ne, en1, wnan;
    int cin, cout;
    if constexpr (kPk) {
      const uint32_t f = r < C ? uint32_t(__double2hiint(a.x)) : 0u;
      ne = f & 1u;
      en1 = (f >> 1) & 1u;
      cin = __double2loint(a.x);
      cout = __double2hiint(b.x);
      wnan = isnan(__int_as_float(__double2loint(b.x)));
    } else {
      ne = !isnan(a.x);
      en1 = b.x == 1.0;
      cin = ne ? int(a.x) : 0;
      cout = ne ? int(a.y) : 0;
      wnan = isnan(b.y);
    }
    int src = -1, dst = -1;
    if (ne) {
      src = tf_lookup(s, cin);
      dst = tf_lookup(s, cout);
    }
    const bool bad = ne && (src < 0 || dst < 0);
    const unsigned m = __ballot_sync(kFull, bad);
    if (m) {
      const int l = __ffs(m) - 1;
      const int ea = __shfl_sync(kFull, ne ? cin : 0, l);
      const int eb = __shfl_sync(kFull, ne ? cout : 0, l);
      if (lane == 0) tf_fail(net, 1 + FNB_E_DANGLING_ENDPOINT, kErrConn, ea, eb, 0);
      return;
    }
    if (r < C) {
      const bool edge = ne && en1;
      uint8_t d = kNoRow;
      if (edge) {
        atomicAdd(&s.R[dst], 1);
        if constexpr (W <= 2) {  // the weight, for step 7 (no re-read of the row)
          if constexpr (kPk) s.cw[r] = __int_as_float(__double2loint(b.x));
          else s.cw[r] = float(b.y);
        }
        if (!wnan) {
          atomicOr(&s.pred[dst * W + (src >> 5)], 1u << (src & 31));
          const int rs = s.rank[src], rd = s.rank[dst];
          atomicOr(&s.predr[rd * W + (rs >> 5)], 1u << (rs & 31));
          d = uint8_t(dst);
        }
      }
      s.csrc[r] = uint8_t(src);
      s.cdst[r] = d;
    }
  }
  __syncwarp();

  // ---- 5. Kahn with min-(key,row) pop (network.hpp:192-214), in rank space:
  //         lane l owns ranks l + 32j.  A rank is ready when every predecessor
  //         has been emitted; the pop is the lowest ready rank (first set bit
  //         of the ready ballots).  Predecessor bits stay in registers for
  //         W <= 4; wider genomes count down with shared-memory bit tests.
  constexpr int NJ = W;  // ranks per lane (N <= 32*W)
  constexpr bool kRegBits = W <= 4;
  uint32_t pr[kRegBits ? NJ : 1][kRegBits ? W : 1];
  int cnt[NJ];
  unsigned live = 0;     // bit j: eligible and not yet emitted
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int rk = lane + 32 * j;
    int pc = 0;
    cnt[j] = 0;
    if (kRegBits) {
#pragma unroll
      for (int w = 0; w < W; ++w) pr[kRegBits ? j : 0][kRegBits ? w : 0] = 0u;
    }
    if (rk < populated) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const uint32_t b = s.predr[rk * W + w];
        pc += __popc(b);
        if (kRegBits) pr[kRegBits ? j : 0][kRegBits ? w : 0] = b;
      }
      const int R = s.R[s.row_of_rank[rk]];
      if (R == pc && (s.sorted_key[rk] >= 0 || R > 0)) live |= 1u << j;
      cnt[j] = pc;
    }
  }
  uint32_t em[W];
#pragma unroll
  for (int w = 0; w < W; ++w) em[w] = 0u;
  int count = 0;
  for (;;) {
    int best = -1;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      bool rdy;
      if (kRegBits) {
        uint32_t pend = 0u;
#pragma unroll
        for (int w = 0; w < W; ++w) pend |= pr[kRegBits ? j : 0][kRegBits ? w : 0] & ~em[w];
        rdy = ((live >> j) & 1u) && pend == 0u;
      } else {
        rdy = ((live >> j) & 1u) && cnt[j] == 0;
      }
      const unsigned b = __ballot_sync(kFull, rdy);
      if (best < 0 && b) best = 32 * j + __ffs(b) - 1;
    }
    if (best < 0) break;
    if (lane == 0) s.order[count] = uint16_t(best);  // a rank; rows below
    ++count;
    const int bw = best >> 5;
    const uint32_t bb = 1u << (best & 31);
    if ((best & 31) == lane) live &= ~(1u << bw);
    if (kRegBits) {
#pragma unroll
      for (int w = 0; w < W; ++w) em[w] |= (w == bw) ? bb : 0u;
    } else {
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        if (((live >> j) & 1u) && (s.predr[(lane + 32 * j) * W + bw] & bb)) --cnt[j];
    }
  }
  __syncwarp();
  uint16_t* gorder = reinterpret_cast<uint16_t*>(net + L.order_off);
  for (int p = lane; p < count; p += 32) {
    const uint16_t row = s.row_of_rank[s.order[p]];
    s.order[p] = row;
    gorder[p] = row;
  }
  __syncwarp();
  if (count != populated) {  // network.hpp:216-218; path rebuilt by k_describe
    if (lane == 0) tf_fail(net, 1 + FNB_E_CYCLE_DETECTED, kErrCycle, 0, 0, count);
    return;
  }

  // ---- 6a. ops in topological order, skipping input rows (network.hpp:252-254):
  //          op index and record base per row; each op = max(1, ceil(fanin/4))
  //          records.  (rank / row_of_rank / R / sorted_key / predr are free
  //          after Kahn and reused as opos / slot_of / last_use / fanin / slot scratch.)
  uint16_t* opos = s.rank;
  uint16_t* slot_of = s.row_of_rank;
  int* last_use = s.R;
  int* fanin = s.sorted_key;
  int op_base = 0, rec_base = 0, edge_total = 0;
  for (int p0 = 0; p0 < count; p0 += 32) {
    const int p = p0 + lane;
    int row = 0, ne = 0, nrec = 0;
    bool is_op = false;
    if (p < count) {
      row = s.order[p];
      is_op = !(s.flags[row] & 2);
      if (is_op) {
#pragma unroll
        for (int w = 0; w < W; ++w) ne += __popc(s.pred[row * W + w]);
        nrec = ne == 0 ? 1 : (ne + kRecSlots - 1) / kRecSlots;
      }
    }
    const unsigned m = __ballot_sync(kFull, is_op);
    int incl = nrec, incl_e = ne;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, d);
      const int te = __shfl_up_sync(kFull, incl_e, d);
      if (lane >= d) { incl += t; incl_e += te; }
    }
    if (is_op) {
      const int k = op_base + __popc(m & ((1u << lane) - 1u));
      opos[row] = uint16_t(k);
      s.op_row[k] = uint16_t(row);
      s.ebeg[row] = uint16_t(rec_base + incl - nrec);
      fanin[row] = ne;
    }
    op_base += __popc(m);
    rec_base += __shfl_sync(kFull, incl, 31);
    edge_total += __shfl_sync(kFull, incl_e, 31);
  }
  // ---- 6b. last consumer (op index) of every value; outputs live to the end
  for (int r = lane; r < N; r += 32) {
    last_use[r] = -1;
    slot_of[r] = 0xffff;
  }
  __syncwarp();
  if (my_out >= 0) last_use[my_out] = kLastForever;
  __syncwarp();
  for (int r = lane; r < C; r += 32) {
    const int dst = s.cdst[r];
    if (dst == kNoRow || (s.flags[dst] & 2)) continue;
    atomicMax(&last_use[s.csrc[r]], int(opos[dst]));
  }
  __syncwarp();
  // ---- 6c. value slots (slots = max live values), warp-parallel: an interval
  //          colouring with a FIFO of free slots (below).  Round 1-2 ran the
  //          lowest-free-slot scan on lane 0, one op after another (27% of K1's
  //          instructions and 23% of its stall samples at C2); this form took K1
  //          from 0.102 to 0.090 ms at C2 and 0.73 to 0.62 ms per 20k genomes at C5.
  int n_slots = 0;
  {
    // Warp-parallel form of the same allocation problem.  Values: the distinct
    // input rows (first appearance), then the ops in order; value v starts at
    // time v and ends at Ip + (its last reader's op index) -- freed before that
    // op's own output is placed, as in the scan -- or right after it starts
    // (an op value nobody reads), or never (outputs, inputs nobody reads).
    // The slot count is the maximum overlap M (what the lowest-free-slot scan
    // reaches: both are optimal for intervals), and the slots come from a FIFO
    // of free slots: start s < M takes slot s, start s >= M the slot of the
    // value whose end is the (s - M)-th end event (time order, ties by value
    // index; __match_any_sync ranks each 32-value chunk).  Slot chains are
    // resolved by pointer jumping.  Any valid assignment gives K2 the same
    // arithmetic, so fitness bits do not depend on it.
    constexpr int kInf = 0x7fff;
    int16_t* endt = reinterpret_cast<int16_t*>(s.kr);  // [N] end time (s.kr is dead after step 2)
    int16_t* vrow = endt + N;                            // [N] row of value v
    int* cnt = reinterpret_cast<int*>(vrow + N);         // [N + 2] end-time histogram, then cursors
    int16_t* srcv = reinterpret_cast<int16_t*>(s.predr);  // [N] value of end event e (predr is dead)
    int16_t* par = endt;                                 // [N] slot chains (endt is dead by then)
    const unsigned lt = (1u << lane) - 1u;
    // distinct inputs in order of first appearance (I <= 32)
    const int irow = my_in;
    bool first = lane < sh.I;
    for (int j = 0; j < sh.I; ++j) {
      const int rj = __shfl_sync(kFull, my_in, j);
      if (j < lane && rj == irow) first = false;
    }
    const unsigned fm = __ballot_sync(kFull, first);
    const int Ip = __popc(fm);
    if (first) vrow[__popc(fm & lt)] = int16_t(irow);
    for (int k = lane; k < op_base; k += 32) vrow[Ip + k] = int16_t(s.op_row[k]);
    const int V = Ip + op_base;
    for (int t = lane; t <= V + 1; t += 32) cnt[t] = 0;
    __syncwarp();
    for (int v = lane; v < V; v += 32) {
      const int lu = last_use[vrow[v]];
      int e;
      if (lu == kLastForever) e = kInf;
      else if (lu < 0) e = v < Ip ? kInf : v + 1;
      else e = Ip + lu;
      endt[v] = int16_t(e);
      if (e != kInf) atomicAdd(&cnt[e], 1);
    }
    __syncwarp();
    // cnt[t] -> #ends before t; live(t) = (t + 1) - #ends at or before t
    int carry = 0, mx = 0;
    for (int t0 = 0; t0 <= V; t0 += 32) {
      const int t = t0 + lane;
      const int c = t <= V ? cnt[t] : 0;
      int incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += y;
      }
      if (t <= V) cnt[t] = carry + incl - c;
      if (t < V) mx = max(mx, t + 1 - (carry + incl));
      carry += __shfl_sync(kFull, incl, 31);
    }
    const int M = int(__reduce_max_sync(kFull, unsigned(mx)));
    __syncwarp();
    // end events in (time, value) order: srcv[e-th end] = value
    for (int v0 = 0; v0 < V; v0 += 32) {
      const int v = v0 + lane;
      const int e = v < V ? int(endt[v]) : kInf;
      const unsigned grp = __match_any_sync(kFull, e);
      const int pos = e != kInf ? cnt[e] + __popc(grp & lt) : 0;
      __syncwarp();
      if (e != kInf) {
        srcv[pos] = int16_t(v);
        if ((grp >> lane) == 1u) cnt[e] += __popc(grp);  // the group's highest lane advances the cursor
      }
      __syncwarp();
    }
    // start s < M takes slot s; start s >= M the slot of the (s - M)-th end
    for (int v = lane; v < V; v += 32) par[v] = int16_t(v < M ? v : srcv[v - M]);
    __syncwarp();
    for (;;) {  // pointer jumping to the chain roots (the slots)
      bool changed = false;
      for (int v = lane; v < V; v += 32) {
        const int q = par[v], qq = par[q];
        if (qq != q) {
          par[v] = int16_t(qq);
          changed = true;
        }
      }
      __syncwarp();
      if (!__any_sync(kFull, changed)) break;
    }
    for (int v = lane; v < V; v += 32) slot_of[vrow[v]] = uint16_t(par[v]);
    n_slots = M;
  }
  n_slots = __shfl_sync(kFull, n_slots, 0);
  __syncwarp();
  // ---- 6d. record headers; pad slots read the zero slot n_slots
  Rec* grec = reinterpret_cast<Rec*>(net + L.ops_off);
  for (int k = lane; k < op_base; k += 32) {
    const int row = s.op_row[k];
    const int ne = fanin[row];
    const int nrec = ne == 0 ? 1 : (ne + kRecSlots - 1) / kRecSlots;
    const int rb = s.ebeg[row];
    const uint16_t code = s.ncode[row];
    RecHeader h;
    h.bias = s.nbias[row];
    h.resp = s.nresp[row];
    h.dst = slot_of[row];
    h.act = uint8_t(code & 0xff);
    h.agg = uint8_t(code >> 8);
    h.fanin = uint16_t(ne);
    for (int q = 0; q < nrec; ++q) {
      h.cnt = uint8_t(min(kRecSlots, ne - q * kRecSlots > 0 ? ne - q * kRecSlots : 0));
      h.flags = uint8_t((q == 0 ? kRecFirst : 0) | (q == nrec - 1 ? kRecLast : 0));
      grec[rb + q].h = h;
    }
    Edge z;  // pad slots of the last record: zero weight, the zero slot
    z.w = 0.0f;
    z.src = uint16_t(n_slots);
    z.conn_row = 0xffff;
    for (int q = ne; q < nrec * kRecSlots; ++q) grec[rb + q / kRecSlots].slot[q % kRecSlots] = z;
  }

  // ---- 7. edges: the i-th predecessor (ascending source row) of an op goes
  //         to slot i%4 of its record i/4, reading the source's value slot
  const uint64_t drop = l2_drop();  // the last read of the connection rows
  for (int r = lane; r < C; r += 32) {
    const int dst = s.cdst[r];
    if (dst == kNoRow || (s.flags[dst] & 2)) continue;
    float wf;
    if constexpr (W <= 2) wf = s.cw[r];
    else wf = kPk ? reinterpret_cast<const float*>(pg + pk.w)[r] : float(ld_l2(crow + r * kConnCols + kW, drop));
    const int src = s.csrc[r];
    int below = 0;
    const int sw = src >> 5;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t bits = s.pred[dst * W + w];
      if (w < sw) below += __popc(bits);
      else if (w == sw) below += __popc(bits & ((1u << (src & 31)) - 1u));
    }
    Edge e;
    e.w = wf;
    e.src = slot_of[src];
    e.conn_row = uint16_t(r);
    grec[s.ebeg[dst] + below / kRecSlots].slot[below % kRecSlots] = e;
  }
  __syncwarp();
  // ---- 8. input / output rows become value slots for the forward
  if (lane < sh.I) in_rows[lane] = slot_of[my_in];
  if (lane < sh.O) out_rows[lane] = slot_of[my_out];
  if (lane == 0) {
    NetHeader* h = reinterpret_cast<NetHeader*>(net);
    h->n_slots = n_slots;
    h->status = 0;
    h->err_kind = kErrNone;
    h->err_a = 0;
    h->err_b = 0;
    h->order_count = int16_t(count);
    h->n_ops = int16_t(op_base);
    h->n_edges = int16_t(edge_total);
    h->n_rec = int16_t(rec_base);
  }
}

// describe_cycle (network.hpp:73-115) for one failing genome, one thread.
// Emitted rows = the partial order K1 stored.  Writes the key path
// (path[0] = length) for the host to format "k1->k2->...->k1".
__global__ void k_describe_cycle(const double* __restrict__ nodes, const double* __restrict__ conns,
                                 const uint8_t* __restrict__ net, NetLayout L, int* path_out) {
  if (threadIdx.x != 0) return;
  const int N = L.N, C = L.C;
  const NetHeader* h = reinterpret_cast<const NetHeader*>(net);
  const uint16_t* order = reinterpret_cast<const uint16_t*>(net + L.order_off);
  uint32_t emitted[(FNB_MAX_NODES_LIMIT + 32) / 32] = {0};
  for (int i = 0; i < h->order_count; ++i) emitted[order[i] >> 5] |= 1u << (order[i] & 31);
  auto empty = [&](int r) { return isnan(nodes[r * kNodeCols]); };
  auto key_of = [&](int r) { return int(nodes[r * kNodeCols]); };
  auto is_em = [&](int r) { return (emitted[r >> 5] >> (r & 31)) & 1u; };
  int start = -1;
  for (int r = 0; r < N; ++r)
    if (!empty(r) && !is_em(r) && (start < 0 || key_of(r) < key_of(start))) start = r;
  if (start < 0) { path_out[0] = -1; return; }
  int16_t pos[FNB_MAX_NODES_LIMIT + 1];
  for (int r = 0; r < N; ++r) pos[r] = -1;
  int len = 0;
  int at = start;
  for (;;) {
    if (pos[at] >= 0) {
      int n = 0;
      for (int i = pos[at]; i < len; ++i) path_out[1 + n++] = path_out[1 + i];
      path_out[1 + n++] = key_of(at);
      path_out[0] = n;
      return;
    }
    pos[at] = int16_t(len);
    path_out[1 + len++] = key_of(at);
    int next = -1;
    for (int r = 0; r < C; ++r) {
      const double* row = conns + size_t(r) * kConnCols;
      if (isnan(row[kIn]) || row[kEn] != 1.0 || int(row[kIn]) != key_of(at)) continue;
      for (int rr = 0; rr < N; ++rr) {
        if (empty(rr) || is_em(rr)) continue;
        if (key_of(rr) == int(row[kOut]) && (next < 0 || key_of(rr) < key_of(next))) next = rr;
      }
    }
    if (next < 0) { path_out[0] = -1; return; }
    at = next;
  }
}

// Lowest failing genome: atomicMin over statuses in the net headers.
__global__ void k_first_error(const uint8_t* __restrict__ nets, size_t stride, int P, int* out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P) return;
  if (reinterpret_cast<const NetHeader*>(nets + size_t(g) * stride)->status != 0) atomicMin(out, g);
}

// int32 order (-1 padded) for parity checks and the host API (network.hpp:32).
__global__ void k_net_order(const uint8_t* __restrict__ nets, NetLayout L, int P,
                            int32_t* __restrict__ order, int32_t* __restrict__ count) {
  const int g = blockIdx.x;
  if (g >= P) return;
  const uint8_t* net = nets + size_t(g) * L.bytes;
  const NetHeader* h = reinterpret_cast<const NetHeader*>(net);
  const uint16_t* o = reinterpret_cast<const uint16_t*>(net + L.order_off);
  const int n = h->status == 0 ? h->order_count : 0;
  for (int i = threadIdx.x; i < L.N; i += blockDim.x)
    if (order) order[size_t(g) * L.N + i] = i < n ? int32_t(o[i]) : -1;
  if (threadIdx.x == 0 && count) count[g] = n;
}

// ---- host launchers --------------------------------------------------------

template <int W, bool kPk>
static cudaError_t launch_transform_w(const double* n, const double* c, const uint8_t* pk, int P, uint8_t* nets,
                                      const NetLayout& L, const DevShape& sh, cudaStream_t st) {
  const size_t per_warp = tf_smem_bytes(sh.N, sh.C, W);
  // CTA width (measured, round 2): 2 warps at N <= 64 (C2 0.104 -> 0.102 ms),
  // 4 above (C5: 0.72 ms per 20k genomes against 0.76 / 0.73 for 2 / 1)
  const int warps = warps_per_cta_for_smem(per_warp, W <= 2 ? 2 : 4);
  const size_t smem = per_warp * warps;
  cudaError_t e = cudaFuncSetAttribute(k_transform<W, kPk>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  const int blocks = (P + warps - 1) / warps;
  k_transform<W, kPk><<<blocks, 32 * warps, smem, st>>>(n, c, pk, P, nets, L, sh, per_warp);
  return cudaGetLastError();
}

template <bool kPk>
static cudaError_t launch_transform_any(const double* n, const double* c, const uint8_t* pk, int P, uint8_t* nets,
                                        const NetLayout& L, const DevShape& sh, cudaStream_t st) {
  const int W = (sh.N + 31) / 32;
  if (W <= 1) return launch_transform_w<1, kPk>(n, c, pk, P, nets, L, sh, st);
  if (W <= 2) return launch_transform_w<2, kPk>(n, c, pk, P, nets, L, sh, st);
  if (W <= 4) return launch_transform_w<4, kPk>(n, c, pk, P, nets, L, sh, st);
  return launch_transform_w<8, kPk>(n, c, pk, P, nets, L, sh, st);
}

cudaError_t launch_transform(const double* n, const double* c, int P, uint8_t* nets, const NetLayout& L,
                             const DevShape& sh, cudaStream_t st) {
  return launch_transform_any<false>(n, c, nullptr, P, nets, L, sh, st);
}

// K1 over packed transfer rows (PackedLayout blocks, one per genome)
cudaError_t launch_transform_packed(const uint8_t* packed, int P, uint8_t* nets, const NetLayout& L,
                                    const DevShape& sh, cudaStream_t st) {
  return launch_transform_any<true>(nullptr, nullptr, packed, P, nets, L, sh, st);
}

cudaError_t launch_describe_cycle(const double* n, const double* c, const uint8_t* net, const NetLayout& L,
                                  int* path, cudaStream_t st) {
  k_describe_cycle<<<1, 32, 0, st>>>(n, c, net, L, path);
  return cudaGetLastError();
}

cudaError_t launch_first_error(const uint8_t* nets, size_t stride, int P, int* out, cudaStream_t st) {
  k_first_error<<<(P + 255) / 256, 256, 0, st>>>(nets, stride, P, out);
  return cudaGetLastError();
}

cudaError_t launch_net_order(const uint8_t* nets, const NetLayout& L, int P, int32_t* order, int32_t* count,
                             cudaStream_t st) {
  k_net_order<<<P, 128, 0, st>>>(nets, L, P, order, count);
  return cudaGetLastError();
}

}  // namespace fnb
