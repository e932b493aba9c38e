// forward.cu -- K2: population x sample-batch forward with fused fitness
// (forward_into / batch_forward, network.hpp:238-330; func-fit and XOR
// fitness) on sm_100a CUDA cores.
//
// Mapping.  A "group" of T threads evaluates one genome over a tile of
// TC = T*SPT sample columns; each thread owns SPT ADJACENT columns so one
// 4/8/16-byte LDS fetches all of its values of a source node.  Node values
// live in shared memory as v[row][TC] (+ one all-zero row); consecutive
// threads touch consecutive 4*SPT-byte chunks, so the irregular per-edge
// source rows never bank-conflict.
//
// Program.  K1 emits each node op as records of exactly four edge slots
// (ascending source row; pad slots carry w = 0 and read the zero row).  The
// records are staged once per CTA with source/destination rows rewritten
// into byte offsets, and the hot loop walks them branch-free: three
// broadcast LDS.128 for the record (prefetched one record ahead), four value
// loads, the FMA chain, and a warp-uniform finalize (activation + store) on
// an op's last record.  A thread only touches its own columns, so the loop
// has no barriers.  Schemas with a single activation/aggregation (the paper
// default {tanh},{sum}) get an instantiation without per-op dispatch.
// Arithmetic is FP32 (north star: 1e-5 relative to the FP64 reference); the
// squared-error fitness accumulates in FP64.
#include <algorithm>
#include <cstdlib>

#include "fnb_common.cuh"

#ifndef FNB_K2_UNROLL
#define FNB_K2_UNROLL 8
#endif
#ifndef FNB_K2_UNROLL_GENERIC
#define FNB_K2_UNROLL_GENERIC 2
#endif

namespace fnb {

// ---- activations (functions.hpp:17-21) in FP32 -----------------------------
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// tanh(x) = 1 - 2/(exp(2x)+1): absolute error ~2e-7 on the whole line,
// saturating exactly to +-1 (inf/0 out of ex2).  Near 0 the form cancels, so
// the error is absolute (~6e-8), not relative: the forward's contract is
// rtol 1e-5 + atol 1e-5 against the FP64 reference.  A
// Taylor branch for |x| < 0.3 made it relative but cost 11% of K2 (0.657 ->
// 0.729 ms at C2), and the FP32 edge sums before it carry the same absolute
// error for outputs near 0 anyway.
__device__ __forceinline__ float tanh_fast(float x) {
  return fmaf(-2.0f, rcp_approx(ex2_approx(x * 2.8853900817779268f) + 1.0f), 1.0f);
}
__device__ __forceinline__ float sigmoid_fast(float x) {
  return rcp_approx(1.0f + ex2_approx(x * -1.4426950408889634f));
}

template <int ACT>
__device__ __forceinline__ float act_apply(int code, float x) {
  const int c = ACT >= 0 ? ACT : code;
  switch (c) {
    case FNB_ACT_IDENTITY: return x;
    case FNB_ACT_TANH: return tanh_fast(x);
    case FNB_ACT_SIGMOID: return sigmoid_fast(x);
    case FNB_ACT_RELU: return x > 0.0f ? x : 0.0f;
    // MUFU.SIN's absolute error grows with |x| (~2^-22 |x|): inside |x| < 32 it
    // stays below 1e-5 (the forward's atol); outside, the accurate sinf
    case FNB_ACT_SIN: return fabsf(x) < 32.0f ? __sinf(x) : sinf(x);
  }
  return x;
}

// ---- staged record (32 B, two float4) ---------------------------------------
//   a = {bias, resp, meta, srcs}   meta = dst | valid << 8 | first << 12 | last << 13
//                                         | act << 16 | agg << 19 | fanin << 21
//                                  valid = one bit per real edge slot; the slot
//                                  bits and first / last share byte 1, so one
//                                  R2P sets all six predicates
//                                  srcs = four u8 source rows (row N = zero row)
//   w = {w0, w1, w2, w3}
struct SRec {
  float4 a, w;
};
static_assert(sizeof(SRec) == 32, "staged record");

template <int SPT> struct VecT;
template <> struct VecT<1> { using T = float; };
template <> struct VecT<2> { using T = float2; };
template <> struct VecT<4> { using T = float4; };

template <int SPT>
__device__ __forceinline__ void vload(const uint8_t* base, uint32_t off, float (&x)[SPT]) {
  const auto v = *reinterpret_cast<const typename VecT<SPT>::T*>(base + off);
  if constexpr (SPT == 1) { x[0] = v; }
  else if constexpr (SPT == 2) { x[0] = v.x; x[1] = v.y; }
  else { x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w; }
}
template <int SPT>
__device__ __forceinline__ void vstore(uint8_t* base, uint32_t off, const float (&x)[SPT]) {
  auto* p = reinterpret_cast<typename VecT<SPT>::T*>(base + off);
  if constexpr (SPT == 1) { *p = x[0]; }
  else if constexpr (SPT == 2) { *p = make_float2(x[0], x[1]); }
  else { *p = make_float4(x[0], x[1], x[2], x[3]); }
}

// Value-row traffic of the hot loop goes through volatile PTX so loads and
// stores stay in program order (a node's result is read by later records),
// and so pad-slot loads can be predicated off: a warp-uniform false
// predicate issues the instruction but moves no shared-memory wavefronts.
template <int SPT>
__device__ __forceinline__ void lds_pred(bool p, uint32_t addr, float (&x)[SPT]) {
  if constexpr (SPT == 1) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %1, 0; @q ld.shared.f32 %0, [%2]; }"
                 : "+f"(x[0]) : "r"(int(p)), "r"(addr));
  } else if constexpr (SPT == 2) {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.shared.v2.f32 {%0, %1}, [%3]; }"
                 : "+f"(x[0]), "+f"(x[1]) : "r"(int(p)), "r"(addr));
  } else {
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %4, 0; @q ld.shared.v4.f32 {%0, %1, %2, %3}, [%5]; }"
                 : "+f"(x[0]), "+f"(x[1]), "+f"(x[2]), "+f"(x[3]) : "r"(int(p)), "r"(addr));
  }
}
// the same with the predicate bit B of `word` (a single LOP3 into a predicate)
template <int SPT, uint32_t B>
__device__ __forceinline__ void lds_bit(uint32_t word, uint32_t addr, float (&x)[SPT]) {
  if constexpr (SPT == 1) {
    asm volatile("{ .reg .pred q; .reg .b32 t; and.b32 t, %1, %2; setp.ne.b32 q, t, 0; @q ld.shared.f32 %0, [%3]; }"
                 : "+f"(x[0]) : "r"(word), "n"(B), "r"(addr));
  } else if constexpr (SPT == 2) {
    asm volatile("{ .reg .pred q; .reg .b32 t; and.b32 t, %2, %3; setp.ne.b32 q, t, 0; @q ld.shared.v2.f32 {%0, %1}, [%4]; }"
                 : "+f"(x[0]), "+f"(x[1]) : "r"(word), "n"(B), "r"(addr));
  } else {
    asm volatile("{ .reg .pred q; .reg .b32 t; and.b32 t, %4, %5; setp.ne.b32 q, t, 0; "
                 "@q ld.shared.v4.f32 {%0, %1, %2, %3}, [%6]; }"
                 : "+f"(x[0]), "+f"(x[1]), "+f"(x[2]), "+f"(x[3]) : "r"(word), "n"(B), "r"(addr));
  }
}
template <int SPT>
__device__ __forceinline__ void sts(uint32_t addr, const float (&x)[SPT]) {
  if constexpr (SPT == 1) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(x[0]));
  } else if constexpr (SPT == 2) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(x[0]), "f"(x[1]));
  } else {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(x[0]), "f"(x[1]), "f"(x[2]),
                 "f"(x[3]));
  }
}

// Packed FP32 pair FMA (FFMA2 on sm_100a): each half is one fma.rn.f32, so
// results are bit-identical to scalar fmaf; the weight is a scalar operand
// broadcast to both halves (no pair construction in SASS).
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpk2(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long ffma2(float w, unsigned long long x, unsigned long long a) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(w, w)), "l"(x), "l"(a));
  return d;
}

struct FwdParams {
  const uint8_t* nets;
  NetLayout L;
  int P;
  const float* X;       // [B][I]
  const float* Y;       // [B][O] or null
  int B;
  int T;                // threads per genome group (power of two)
  int groups;           // genome groups per CTA (threads beyond groups*T idle)
  int fit_kind;
  double fit_offset;
  double* fitness;      // [P] or null
  double* out;          // [P][B][O] or null
  double* partial;      // [P][units]: squared error of each 32-sample unit
  int units;            // ceil(B / 32)
  size_t group_smem;    // bytes per group
  // this pass evaluates genomes that fit (n_slots + 1 <= rows_hi value rows and
  // n_rec + 1 <= recs_hi records) and, for the overflow pass, do not fit the
  // main pass's (prev_rows, prev_recs); prev_rows = 0 in the main pass
  int rows_hi, recs_hi, prev_rows, prev_recs;
  uint32_t rec_bytes;   // record area of a group (recs_hi records, 16-byte aligned)
};

__host__ __device__ inline size_t fwd_group_smem(int N, int C, int I, int O, int T, int spt, int rows, int recs) {
  size_t b = align16(size_t(recs) * sizeof(SRec));  // records + the zero sentinel
  b += align16(size_t(I + O) * sizeof(uint32_t));
  b += size_t(rows) * size_t(T) * spt * sizeof(float);      // value slots + zero slot
  return align16(b);
}

template <int SPT, int AGG, int ACT>
__global__ void __launch_bounds__(256)
k_forward(FwdParams p) {
  constexpr bool kBounded = ACT == FNB_ACT_TANH || ACT == FNB_ACT_SIGMOID;
  // {sum} schemas: the accumulators are reset at each finalize instead of on
  // each op's first record
  constexpr bool kSumOnly = AGG == FNB_AGG_SUM;
  // record loop unrolling: the single-function instantiations gain from a
  // deeper unroll (more independent record bodies in flight), the generic
  // one (activation / aggregation dispatch per op) does not
  constexpr int kRecUnroll = (AGG >= 0 && ACT >= 0) ? FNB_K2_UNROLL : FNB_K2_UNROLL_GENERIC;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int T = p.T;
  const int grp = threadIdx.x / T;
  const int j = threadIdx.x % T;
  const int g = blockIdx.x * p.groups + grp;
  const NetLayout& L = p.L;
  uint8_t* base = smem_raw + size_t(grp < p.groups ? grp : 0) * p.group_smem;
  SRec* s_rec = reinterpret_cast<SRec*>(base);
  uint32_t* s_io = reinterpret_cast<uint32_t*>(base + p.rec_bytes);
  uint8_t* v = reinterpret_cast<uint8_t*>(s_io) + align16(size_t(L.I + L.O) * sizeof(uint32_t));
  const int TC = T * SPT;                                 // columns per tile
  const uint32_t row_shift = uint32_t(__ffs(TC * 4) - 1);  // v row stride = TC*4 bytes (a power of two)
  const uint32_t row_bytes = uint32_t(TC) * 4u;
  const uint32_t vb = uint32_t(__cvta_generic_to_shared(v)) + uint32_t(j) * SPT * 4u;  // my columns

  bool live = grp < p.groups && g < p.P;
  int n_rec = 0, n_slots = 0;
  if (live) {  // genomes needing more value rows or records than the main pass holds go to the overflow pass
    const NetHeader* hd = reinterpret_cast<const NetHeader*>(p.nets + size_t(g) * L.bytes);
    n_slots = hd->n_slots;
    const int nr = hd->n_rec;
    const bool fits = n_slots + 1 <= p.rows_hi && nr + 1 <= p.recs_hi;
    const bool fits_main = n_slots + 1 <= p.prev_rows && nr + 1 <= p.prev_recs;
    live = hd->status == 0 && fits && (p.prev_rows == 0 || !fits_main);
  }
  if (live) {
    const uint8_t* net = p.nets + size_t(g) * L.bytes;
    n_rec = reinterpret_cast<const NetHeader*>(net)->n_rec;
    const Rec* gr = reinterpret_cast<const Rec*>(net + L.ops_off);
    for (int i = j; i < n_rec; i += T) {
      const Rec r = gr[i];
      const uint32_t meta = uint32_t(r.h.dst) | (((1u << r.h.cnt) - 1u) << 8) | (uint32_t(r.h.flags) << 12) |
                            (uint32_t(r.h.act) << 16) | (uint32_t(r.h.agg) << 19) | (uint32_t(r.h.fanin) << 21);
      const uint32_t srcs = uint32_t(r.slot[0].src) | (uint32_t(r.slot[1].src) << 8) |
                            (uint32_t(r.slot[2].src) << 16) | (uint32_t(r.slot[3].src) << 24);
      s_rec[i] = SRec{make_float4(r.h.bias, r.h.resp, __uint_as_float(meta), __uint_as_float(srcs)),
                      make_float4(r.slot[0].w, r.slot[1].w, r.slot[2].w, r.slot[3].w)};
    }
    if (j == 0) s_rec[n_rec] = SRec{make_float4(0, 0, 0, 0), make_float4(0, 0, 0, 0)};
    const uint16_t* sio = reinterpret_cast<const uint16_t*>(net + L.in_off);
    for (int i = j; i < L.I + L.O; i += T) s_io[i] = uint32_t(sio[i]) << row_shift;
    float z[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) z[k] = 0.0f;
    sts<SPT>(vb + (uint32_t(n_slots) << row_shift), z);  // the all-zero pad slot
  }
  __syncthreads();

  const int I = L.I, O = L.O;
  const bool vec_x = (reinterpret_cast<uintptr_t>(p.X) & 15) == 0;
  // fitness units: 32 consecutive samples, reduced by an adjacent-pair tree
  // (in-thread over SPT, then shfl_xor over the unit's lanes); samples >= B
  // add exact zeros, so a unit's sum depends on neither T, SPT, the chunking
  // nor the population it is evaluated with
  const int ulanes = min(32 / SPT, T);
  const int lane = threadIdx.x & 31;
  const unsigned gmask = T >= 32 ? 0xffffffffu : (((1u << T) - 1u) << (lane & ~(T - 1)));
  // sample tiles of this CTA's y-chunk; dead groups (g >= P) run zero tiles
  // but stay resident for the warp-synchronous reduction below
  const int tiles = (p.B + TC - 1) / TC;
  const int per = (tiles + gridDim.y - 1) / gridDim.y;
  const int t_lo = blockIdx.y * per;
  const int t_hi = live ? min(tiles, t_lo + per) : t_lo;
  for (int tile = t_lo; tile < t_hi; ++tile) {
    const int s0 = tile * TC + j * SPT;  // first sample of this thread
    // seed input rows (network.hpp:249-250).  A thread's SPT samples are
    // SPT*I consecutive floats of X; with I = 4 they are read as SPT float4
    // (two lines per warp-instruction instead of eight scalar loads' worth)
    if (I == 4 && s0 + SPT <= p.B && vec_x) {
      const float4* xs = reinterpret_cast<const float4*>(p.X + size_t(s0) * 4);
      float4 v[SPT];
#pragma unroll
      for (int k = 0; k < SPT; ++k) v[k] = __ldg(xs + k);
      float x[SPT];
#pragma unroll
      for (int k = 0; k < SPT; ++k) x[k] = v[k].x;
      sts<SPT>(vb + s_io[0], x);
#pragma unroll
      for (int k = 0; k < SPT; ++k) x[k] = v[k].y;
      sts<SPT>(vb + s_io[1], x);
#pragma unroll
      for (int k = 0; k < SPT; ++k) x[k] = v[k].z;
      sts<SPT>(vb + s_io[2], x);
#pragma unroll
      for (int k = 0; k < SPT; ++k) x[k] = v[k].w;
      sts<SPT>(vb + s_io[3], x);
    } else {
      for (int i = 0; i < I; ++i) {
        float x[SPT];
#pragma unroll
        for (int k = 0; k < SPT; ++k) x[k] = (s0 + k < p.B) ? __ldg(p.X + size_t(s0 + k) * I + i) : 0.0f;
        sts<SPT>(vb + s_io[i], x);
      }
    }
    // ops in topological order (network.hpp:252-264), one record per step.
    // cur.w is reloaded once this record's FMAs are done; the header (meta,
    // source rows, bias / response) two records ahead, so its fetch overlaps
    // a whole record (C5 4.73 -> 4.45 ms per 20k genomes; the weights two
    // ahead as well measured slower, 4.68 ms).
    float acc[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) acc[k] = 0.0f;
    SRec cur = s_rec[0];
    // the record header two ahead is in flight a whole record body (its
    // meta / source rows start the next-but-one record's dependency chain)
    float4 a_next = s_rec[n_rec > 0 ? 1 : 0].a;
    float x0[SPT], x1[SPT], x2[SPT], x3[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) x0[k] = x1[k] = x2[k] = x3[k] = 0.0f;
#pragma unroll kRecUnroll
    for (int r = 0; r < n_rec; ++r) {
      const uint32_t meta = __float_as_uint(cur.a.z);
      const uint32_t srcs = __float_as_uint(cur.a.w);
      const bool first = (meta >> 12) & 1u;
      const bool last = (meta >> 13) & 1u;
      const int agg = AGG >= 0 ? AGG : int((meta >> 19) & 3u);
      // pad slots are predicated off (no shared-memory traffic; their weight
      // is 0).  With a bounded activation every value a slot register can
      // hold (an input, a node value, 0) is finite, so a pad slot's stale
      // operand contributes 0 * x = +-0 and the registers need no zeroing;
      // otherwise (identity / relu could overflow to inf) they are zeroed.
      if (!kBounded) {
#pragma unroll
        for (int k = 0; k < SPT; ++k) x0[k] = x1[k] = x2[k] = x3[k] = 0.0f;
      }
      // one PRMT (byte extract) + one IMAD (row address) per slot
      lds_bit<SPT, 1u << 8>(meta, vb + __byte_perm(srcs, 0u, 0x4440) * row_bytes, x0);
      lds_bit<SPT, 1u << 9>(meta, vb + __byte_perm(srcs, 0u, 0x4441) * row_bytes, x1);
      lds_bit<SPT, 1u << 10>(meta, vb + __byte_perm(srcs, 0u, 0x4442) * row_bytes, x2);
      lds_bit<SPT, 1u << 11>(meta, vb + __byte_perm(srcs, 0u, 0x4443) * row_bytes, x3);
      if (agg == FNB_AGG_SUM || agg == FNB_AGG_MEAN) {
        // pad slots contribute 0 * 0: branch-free, ascending source row
if constexpr (SPT == 1) {
          float a = (kSumOnly || !first) ? acc[0] : 0.0f;
          a = fmaf(cur.w.x, x0[0], a);
          a = fmaf(cur.w.y, x1[0], a);
          a = fmaf(cur.w.z, x2[0], a);
          a = fmaf(cur.w.w, x3[0], a);
          acc[0] = a;
        } else {
#pragma unroll
          for (int k = 0; k < SPT; k += 2) {
            unsigned long long a = (kSumOnly || !first) ? pk2(acc[k], acc[k + 1]) : 0ull;
            a = ffma2(cur.w.x, pk2(x0[k], x0[k + 1]), a);
            a = ffma2(cur.w.y, pk2(x1[k], x1[k + 1]), a);
            a = ffma2(cur.w.z, pk2(x2[k], x2[k + 1]), a);
            a = ffma2(cur.w.w, pk2(x3[k], x3[k + 1]), a);
            unpk2(a, acc[k], acc[k + 1]);
          }
        }
      } else {
        const int cnt = __popc((meta >> 8) & 15u);  // real slots are a prefix
        const float w[4] = {cur.w.x, cur.w.y, cur.w.z, cur.w.w};
        if (agg == FNB_AGG_PRODUCT) {  // one (warp-uniform) branch per record, not per sample
#pragma unroll
          for (int k = 0; k < SPT; ++k) {
            const float xs[4] = {x0[k], x1[k], x2[k], x3[k]};
            float a = first ? 1.0f : acc[k];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q < cnt) a *= w[q] * xs[q];
            acc[k] = a;
          }
        } else {  // max; empty fan-in falls back to 0 (network.hpp:258-261)
#pragma unroll
          for (int k = 0; k < SPT; ++k) {
            const float xs[4] = {x0[k], x1[k], x2[k], x3[k]};
            float a = first ? 0.0f : acc[k];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float t = w[q] * xs[q];
              if (q < cnt) a = ((first && q == 0) || t > a) ? t : a;
            }
            acc[k] = a;
          }
        }
      }
      cur.w = s_rec[r + 1].w;
      if (last) {
        if (agg == FNB_AGG_MEAN) {
          const uint32_t fanin = meta >> 21;
          if (fanin > 0) {
            const float rn = rcp_approx(float(fanin));  // fanin <= 255: rcp.approx is within 1 ulp
#pragma unroll
            for (int k = 0; k < SPT; ++k) acc[k] = acc[k] * rn;
          }
        }
        float y[SPT];
        if constexpr (ACT >= 0) {
#pragma unroll
          for (int k = 0; k < SPT; ++k) y[k] = act_apply<ACT>(ACT, fmaf(cur.a.y, acc[k], cur.a.x));
        } else {  // one dispatch per op (warp-uniform), not per sample
#pragma unroll
          for (int k = 0; k < SPT; ++k) y[k] = fmaf(cur.a.y, acc[k], cur.a.x);
          switch (int((meta >> 16) & 7u)) {
            case FNB_ACT_TANH:
#pragma unroll
              for (int k = 0; k < SPT; ++k) y[k] = tanh_fast(y[k]);
              break;
            case FNB_ACT_SIGMOID:
#pragma unroll
              for (int k = 0; k < SPT; ++k) y[k] = sigmoid_fast(y[k]);
              break;
            case FNB_ACT_RELU:
#pragma unroll
              for (int k = 0; k < SPT; ++k) y[k] = y[k] > 0.0f ? y[k] : 0.0f;
              break;
            case FNB_ACT_SIN:
#pragma unroll
              for (int k = 0; k < SPT; ++k) y[k] = act_apply<FNB_ACT_SIN>(FNB_ACT_SIN, y[k]);
              break;
            default: break;  // identity
          }
        }
        sts<SPT>(vb + (meta & 0xffu) * row_bytes, y);
        if constexpr (kSumOnly) {
#pragma unroll
          for (int k = 0; k < SPT; ++k) acc[k] = 0.0f;  // the next op starts from 0
        }
      }
      cur.a = a_next;
      a_next = s_rec[min(r + 2, n_rec)].a;
    }
    // outputs + fitness epilogue: per-sample squared error, outputs in order
    double e[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) e[k] = 0.0;
    for (int o = 0; o < O; ++o) {
      float val[SPT];
      lds_pred<SPT>(true, vb + s_io[I + o], val);
#pragma unroll
      for (int k = 0; k < SPT; ++k) {
        const int s = s0 + k;
        if (s >= p.B) continue;
        if (p.out) p.out[(size_t(g) * p.B + s) * O + o] = double(val[k]);
        if (p.fit_kind != FNB_FIT_NONE) {
          const double d = double(__ldg(p.Y + size_t(s) * O + o)) - double(val[k]);
          e[k] += d * d;
        }
      }
    }
    if (p.fit_kind != FNB_FIT_NONE) {
      double u;
      if constexpr (SPT == 1) u = e[0];
      else if constexpr (SPT == 2) u = e[0] + e[1];
      else u = (e[0] + e[1]) + (e[2] + e[3]);
      for (int m = 1; m < ulanes; m <<= 1) u += __shfl_xor_sync(gmask, u, m);
      if ((j & (ulanes - 1)) == 0 && s0 < p.B) p.partial[size_t(g) * p.units + (s0 >> 5)] = u;
    }
  }
}

// fitness = ordered sum of the 32-sample units (network.hpp's evaluate loop
// order is restated in tests/ with a tolerance; the device order is fixed)
__global__ void k_fitness_finalize(const double* __restrict__ partial, int units, int P, int B, int O,
                                   int fit_kind, double offset, double* __restrict__ fitness) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P) return;
  double sse = 0.0;
  for (int c = 0; c < units; ++c) sse += partial[size_t(g) * units + c];
  fitness[g] = fit_kind == FNB_FIT_NEG_MSE ? -(sse / (double(B) * double(O))) : offset - sse;
}

__global__ void k_to_float(const double* __restrict__ src, float* __restrict__ dst, size_t n, int* bad) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = src[i];
  if (!isfinite(x)) atomicOr(bad, 1);
  dst[i] = float(x);
}

// ---- host launchers --------------------------------------------------------

struct FwdConfig {
  int T, spt, block, groups, chunks, grid_x, rows, recs;
  size_t group_smem, cta_smem;
};

static int g_force_spt = 0;       // tuning override (fnb_set_forward_spt)
static int g_rows_pct = 0;        // main-pass slot capacity, % of max_nodes + 1 (0: by shape, main_rows)
static int g_max_cols = 256;      // sample columns per genome group (tile width; swept, scripts/sweep_forward.py)
static int g_group_kb = 72;       // shared-memory budget of one genome group
static int g_recs_pct = 60;       // main-pass record capacity, % of max_records + 1

// Launch geometry for `rows` value rows per column (slots + the zero slot).
static FwdConfig fwd_config(const NetLayout& L, int P, int B, int rows, int recs, bool single_chunk) {
  FwdConfig c{};
  c.rows = rows;
  c.recs = recs;
  // columns per group: cover the batch, at most 256, shrinking until a
  // group fits ~72 KB (>= 3 resident CTAs per SM)
  int cols = 1;
  while (cols < B && cols < g_max_cols) cols <<= 1;
  static const int env_spt = [] {  // experiment knob (fnb_set_forward_spt overrides)
    const char* e = std::getenv("FNB_FWD_SPT");
    return e ? std::atoi(e) : 0;
  }();
  const int force = g_force_spt ? g_force_spt : (env_spt == 1 || env_spt == 2 || env_spt == 4 ? env_spt : 0);
  int spt = force ? force : (cols >= 128 ? 2 : 1);
  while (cols > 32 && fwd_group_smem(L.N, L.C, L.I, L.O, std::max(1, cols / spt), spt, rows, recs) > size_t(g_group_kb) * 1024)
    cols >>= 1;
  spt = std::min(spt, cols);
  const int T = std::max(1, cols / spt);
  c.spt = spt;
  c.T = T;
  c.group_smem = fwd_group_smem(L.N, L.C, L.I, L.O, T, spt, rows, recs);
  // groups per CTA: up to 256 threads, chosen to fit the most groups into an
  // SM's 228 KB (each CTA also reserves 1 KB): at C2 (24.6 KB groups) 1 or 3
  // groups per CTA make 9 resident groups where 2 or 4 make 8
  int groups = 1, best = 0;
  for (int g = 1; g <= std::max(1, 256 / T); ++g) {
    const size_t cta = c.group_smem * size_t(g) + 1024;
    if (cta > 227 * 1024 + 1024) break;
    const int resident = int((228 * 1024) / cta) * g;
    if (resident > best) { best = resident; groups = g; }
  }
  c.groups = groups;
  c.block = std::max(32, groups * T);
  c.cta_smem = c.group_smem * groups;
  c.grid_x = (P + groups - 1) / groups;
  const int tiles = (B + T * spt - 1) / (T * spt);
  const int target = 4 * 148;  // >= 4 CTAs per SM before splitting samples
  c.chunks = 1;
  if (!single_chunk && c.grid_x < target) c.chunks = std::min(tiles, (target + c.grid_x - 1) / c.grid_x);
  static const int force_chunks = [] {  // experiment knob: sample tiles split over blockIdx.y
    const char* e = std::getenv("FNB_FWD_CHUNKS");
    return e ? std::atoi(e) : 0;
  }();
  if (!single_chunk && force_chunks > 0) c.chunks = std::min(tiles, force_chunks);
  return c;
}

// Main-pass capacities (round-2 sweep, scripts/sweep_forward.py and
// scripts/exp_forward_cfg.py, fill-0.75 populations): 62% of the value rows
// at N_max <= 64 (C2: 0.643 -> 0.608 ms together with 256-column tiles and
// 60% of the records) and 72% above (C5: 5.43 -> 5.20 ms per 20k genomes);
// genomes beyond either capacity run in the overflow pass
static int main_rows(const NetLayout& L) {
  const int pct = g_rows_pct ? g_rows_pct : (L.N <= 64 ? 62 : 72);
  return std::min(L.N + 1, std::max(16, ((L.N + 1) * pct + 99) / 100));
}
static int all_recs(const NetLayout& L) { return max_records(L.N, L.C) + 1; }
static int main_recs(const NetLayout& L) {
  return std::min(all_recs(L), std::max(16, (all_recs(L) * g_recs_pct + 99) / 100));
}
void set_forward_recs_pct(int pct) { g_recs_pct = (pct >= 10 && pct <= 100) ? pct : 60; }

void set_forward_spt(int spt) { g_force_spt = (spt == 1 || spt == 2 || spt == 4) ? spt : 0; }
void set_forward_rows_pct(int pct) { g_rows_pct = (pct >= 10 && pct <= 100) ? pct : 0; }
void set_forward_tuning(int spt, int max_cols, int rows_pct, int group_kb) {
  set_forward_spt(spt);
  set_forward_rows_pct(rows_pct);
  g_max_cols = (max_cols >= 32 && max_cols <= 1024 && (max_cols & (max_cols - 1)) == 0) ? max_cols : 256;
  g_group_kb = (group_kb >= 8 && group_kb <= 220) ? group_kb : 72;
}

static int fitness_units(int B) { return (B + 31) / 32; }

size_t forward_partial_needed(NetLayout, int P, int B) {
  return sizeof(double) * size_t(P) * size_t(fitness_units(B)) + 16;
}

cudaError_t launch_to_float(const double* src, float* dst, size_t n, int* bad, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_to_float<<<int((n + 255) / 256), 256, 0, st>>>(src, dst, n, bad);
  return cudaGetLastError();
}

template <int SPT, int AGG, int ACT>
static cudaError_t launch_k(const FwdConfig& c, const FwdParams& p, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k_forward<SPT, AGG, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(c.cta_smem));
  if (e != cudaSuccess) return e;
  // node values are the occupancy limiter: ask for the full 228 KB carveout
  e = cudaFuncSetAttribute(k_forward<SPT, AGG, ACT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           int(cudaSharedmemCarveoutMaxShared));
  if (e != cudaSuccess) return e;
  k_forward<SPT, AGG, ACT><<<dim3(c.grid_x, c.chunks), c.block, c.cta_smem, st>>>(p);
  return cudaGetLastError();
}

template <int SPT>
static cudaError_t launch_spt(const FwdConfig& c, const FwdParams& p, int agg, int act, cudaStream_t st) {
  if (agg == FNB_AGG_SUM) {
    switch (act) {
      case FNB_ACT_TANH: return launch_k<SPT, FNB_AGG_SUM, FNB_ACT_TANH>(c, p, st);
      case FNB_ACT_SIGMOID: return launch_k<SPT, FNB_AGG_SUM, FNB_ACT_SIGMOID>(c, p, st);
      case FNB_ACT_IDENTITY: return launch_k<SPT, FNB_AGG_SUM, FNB_ACT_IDENTITY>(c, p, st);
      case FNB_ACT_RELU: return launch_k<SPT, FNB_AGG_SUM, FNB_ACT_RELU>(c, p, st);
      default: break;
    }
  }
  return launch_k<SPT, -1, -1>(c, p, st);
}

static cudaError_t launch_pass(const FwdConfig& c, FwdParams p, int prev_rows, int prev_recs, int agg, int act,
                               cudaStream_t st) {
  if (c.cta_smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  p.T = c.T;
  p.groups = c.groups;
  p.group_smem = c.group_smem;
  p.rows_hi = c.rows;
  p.recs_hi = c.recs;
  p.prev_rows = prev_rows;
  p.prev_recs = prev_recs;
  p.rec_bytes = uint32_t(align16(size_t(c.recs) * sizeof(SRec)));
  switch (c.spt) {
    case 4: return launch_spt<4>(c, p, agg, act, st);
    case 2: return launch_spt<2>(c, p, agg, act, st);
    default: return launch_spt<1>(c, p, agg, act, st);
  }
}

// Side stream + fork/join events of the overflow pass, per host thread and
// device (a context is used from one host thread; graph capture follows the
// fork into the side stream and back).
struct FwdAux {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static FwdAux& fwd_aux() {
  static thread_local FwdAux aux[64];
  int dev = 0;
  cudaGetDevice(&dev);
  FwdAux& x = aux[dev & 63];
  if (!x.side) {
    if (cudaStreamCreateWithFlags(&x.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess)
      x.side = nullptr;
  }
  return x;
}

// Two passes: genomes whose live values fit the main slot capacity (almost
// all) and -- over the same grid, exiting immediately for the rest, on a side
// stream concurrently -- the few that need up to max_nodes + 1 rows.
// uniform_agg / uniform_act: the single registry entry, or -1 for mixed schemas
int launch_forward(const void* nets, NetLayout L, int P, const float* X, const float* Y, int B, int fit_kind,
                   double offset, double* fitness, double* out, double* partial_buf, size_t partial_cap,
                   int uniform_agg, int uniform_act, cudaStream_t st, long long* launches) {
  const int rows_main = main_rows(L), recs_main = main_recs(L);
  const FwdConfig c = fwd_config(L, P, B, rows_main, recs_main, false);
  FwdParams p;
  p.nets = static_cast<const uint8_t*>(nets);
  p.L = L;
  p.P = P;
  p.X = X;
  p.Y = Y;
  p.B = B;
  p.fit_kind = fit_kind;
  p.fit_offset = offset;
  p.fitness = fitness;
  p.out = out;
  p.partial = partial_buf;
  p.units = fitness_units(B);
  const bool fit = fit_kind != FNB_FIT_NONE;
  if (fit && sizeof(double) * size_t(P) * p.units > partial_cap) return 1;
  if (rows_main < L.N + 1 || recs_main < all_recs(L)) {
    // The overflow pass (a few genomes, long per-CTA latency) runs on a side
    // stream next to the main pass instead of as a tail after it; both write
    // disjoint genomes' units, so no bit depends on the overlap.
    FwdAux& x = fwd_aux();
    if (!x.side) return 1;
    const FwdConfig co = fwd_config(L, P, B, L.N + 1, all_recs(L), true);
    if (cudaEventRecord(x.fork, st) != cudaSuccess || cudaStreamWaitEvent(x.side, x.fork, 0) != cudaSuccess) return 1;
    if (launch_pass(co, p, rows_main, recs_main, uniform_agg, uniform_act, x.side) != cudaSuccess) return 1;
    if (cudaEventRecord(x.join, x.side) != cudaSuccess) return 1;
    if (launch_pass(c, p, 0, 0, uniform_agg, uniform_act, st) != cudaSuccess) return 1;
    if (cudaStreamWaitEvent(st, x.join, 0) != cudaSuccess) return 1;
    *launches += 2;
  } else {
    if (launch_pass(c, p, 0, 0, uniform_agg, uniform_act, st) != cudaSuccess) return 1;
    ++*launches;
  }
  if (fit) {
    k_fitness_finalize<<<(P + 255) / 256, 256, 0, st>>>(partial_buf, p.units, P, B, L.O, fit_kind, offset, fitness);
    if (cudaGetLastError() != cudaSuccess) return 1;
    ++*launches;
  }
  return 0;
}

}  // namespace fnb
