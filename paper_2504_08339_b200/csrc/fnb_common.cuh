// fnb_common.cuh -- device-side layout shared by the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "flatneat_b200.h"

namespace fnb {

// Row layout of the reference tensors (genome.hpp:19-38).
constexpr int kNodeCols = 5, kConnCols = 4;
constexpr int kKey = 0, kBias = 1, kResp = 2, kAgg = 3, kAct = 4;
constexpr int kIn = 0, kOut = 1, kEn = 2, kW = 3;

// Error detail kinds written by K1 next to the status (for the reference
// what() strings of network.hpp:147-178, 216-218).
enum ErrKind : int32_t {
  kErrNone = 0,
  kErrActId = 1,       // "activation id %d out of range"
  kErrAggId = 2,       // "aggregation id %d out of range"
  kErrInputKey = 3,    // "input key %d"
  kErrOutputKey = 4,   // "output key %d"
  kErrConn = 5,        // "conn (%d, %d)"
  kErrCycle = 6,       // "cycle <path>" (path rebuilt by the describe kernel)
};

// ---- transformed network (one fixed-stride block per genome in HBM) ------
// Compact replacement of TransformedNetwork (network.hpp:29-67): the dense
// max_nodes^2 `expanded` tensor is never materialised; each node op carries
// its incoming edges in ascending source row, the accumulation order of
// network.hpp:184-190.
struct NetHeader {          // 32 B
  int32_t status;           // 0 or 1 + Errc
  int32_t err_kind;
  int32_t err_a, err_b;
  int16_t order_count;
  int16_t n_ops;            // non-input rows in order
  int16_t n_edges;          // enabled edges feeding ops
  int16_t n_rec;            // forward records
  int32_t n_slots;          // forward value slots (liveness-shared); slot n_slots = zero row
  int32_t pad2;
};
static_assert(sizeof(NetHeader) == 32, "header");

struct Op {                 // 16 B, one per non-input node in topological order
  float bias;
  float resp;
  uint16_t dst;             // node row
  uint16_t e_begin;
  uint16_t e_end;
  uint8_t act;              // built-in code (fnb_act)
  uint8_t agg;              // built-in code (fnb_agg)
};
static_assert(sizeof(Op) == 16, "op");

struct Edge {               // 8 B
  float w;
  uint16_t src;             // source node row (max_nodes = the all-zero pad row)
  uint16_t conn_row;        // connection row the weight came from (0xffff: pad)
};
static_assert(sizeof(Edge) == 8, "edge");

// Forward program record: one node op split into chunks of four incoming
// edges (ascending source row).  Pad slots have w = 0 and read the extra
// all-zero value row, so the hot loop is branch-free.
constexpr int kRecSlots = 4;
constexpr uint8_t kRecFirst = 1, kRecLast = 2;
struct RecHeader {          // 16 B
  float bias;
  float resp;
  uint16_t dst;             // node row written by the op's last record
  uint8_t cnt;              // real edges in this record (0..4)
  uint8_t flags;            // kRecFirst | kRecLast
  uint8_t act, agg;
  uint16_t fanin;           // op's total fan-in (mean)
};
struct Rec {                // 48 B
  RecHeader h;
  Edge slot[kRecSlots];
};
static_assert(sizeof(RecHeader) == 16 && sizeof(Rec) == 48, "record");
__host__ __device__ inline int max_records(int N, int C) { return N + (C + kRecSlots - 1) / kRecSlots; }

// kernels one K3 distance call launches (distance.cu: 6 union-table build kernels + k_distance)
constexpr int kDistanceLaunches = 7;

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// L2 residency hints (createpolicy + ld.global.L2::cache_hint).  A kernel
// that reads a genome row early, runs a long per-genome phase, and reads the
// row again (K1's weights, K6's weights) loads it evict_last the first time,
// so it is still in L2 at the second access, and evict_first the last time,
// which releases it: the genome crosses HBM once.
#ifdef __CUDACC__
__device__ __forceinline__ uint64_t l2_keep() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_drop() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_l2(const double* a, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld2_l2(const double* a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
  return v;
}
// One TMA bulk prefetch of [a, a + bytes) into L2 (bytes a multiple of 16, a
// 16-byte aligned): a warp that will stream a genome's rows after a long
// shared-memory phase issues it first, so the rows come from L2, not HBM.
__device__ __forceinline__ void prefetch_l2_bulk(const void* a, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
}
// the same for any byte range (widened to 16-byte boundaries)
__device__ __forceinline__ void prefetch_l2_range(const void* a, size_t bytes) {
  const uintptr_t lo = reinterpret_cast<uintptr_t>(a) & ~uintptr_t(15);
  const uintptr_t hi = (reinterpret_cast<uintptr_t>(a) + bytes + 15) & ~uintptr_t(15);
  if (hi > lo) prefetch_l2_bulk(reinterpret_cast<const void*>(lo), uint32_t(hi - lo));
}
#endif

struct NetLayout {
  int N, C, I, O;
  size_t ops_off, edges_off, order_off, in_off, out_off, bytes;
  __host__ __device__ NetLayout() : NetLayout(0, 0, 0, 0) {}
  __host__ __device__ NetLayout(int n, int c, int i, int o) : N(n), C(c), I(i), O(o) {
    ops_off = sizeof(NetHeader);  // forward records (Rec)
    edges_off = ops_off;          // (edges live inside the records)
    order_off = align16(ops_off + size_t(max_records(N, C)) * sizeof(Rec));
    in_off = align16(order_off + size_t(N) * sizeof(uint16_t));
    out_off = in_off + size_t(I) * sizeof(uint16_t);
    bytes = align16(out_off + size_t(O) * sizeof(uint16_t));
  }
};

// Packed transfer rows (the host-buffer evaluate path): what K1 reads of a
// genome, converted on the host exactly as K1 converts the FP64 rows on the
// device (int() truncating, NaN -> INT32_MIN, saturating; float() rounded
// to nearest), structure-of-arrays so every warp load is coalesced.  16N +
// 13C bytes against 40N + 32C (0.40 at C2); node act / agg ids must fit a
// byte (the host packer falls back to the FP64 rows otherwise).
struct PackedLayout {
  size_t key, bias, resp, act, agg, nflag, cin, cout, w, cflag, bytes;
  __host__ __device__ PackedLayout(int N, int C) {
    key = 0;
    bias = 4 * size_t(N);
    resp = 8 * size_t(N);
    act = 12 * size_t(N);
    agg = 13 * size_t(N);
    nflag = 14 * size_t(N);  // bit0: non-empty (key not NaN)
    cin = (15 * size_t(N) + 3) & ~size_t(3);
    cout = cin + 4 * size_t(C);
    w = cout + 4 * size_t(C);
    cflag = w + 4 * size_t(C);  // bit0: non-empty (in not NaN), bit1: enabled == 1.0
    bytes = align16(cflag + size_t(C));
  }
};

// Schema + shape constants passed by value to kernels.
struct DevShape {
  int N, C, I, O;
  int n_act, n_agg;
  uint8_t act[8];
  uint8_t agg[8];
  int default_act, default_agg;
  int input_keys[32];
  int output_keys[32];
};

// Warps per CTA (a power of two <= max_warps) that lets the most warps of a
// warp-per-item kernel reside on an SM when shared memory is what limits it
// (1 KB per CTA is reserved by the hardware).  Ties keep the larger CTA.
inline int warps_per_cta_for_smem(size_t per_warp, int max_warps) {
  static int smem_sm = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    return v > 0 ? v : 233472;
  }();
  int best_w = 1;
  long best = -1;
  for (int w = max_warps; w >= 1; --w) {
    long ctas = long(smem_sm) / long(size_t(w) * per_warp + 1024);
    if (ctas > 32) ctas = 32;
    if (ctas * w > best) {
      best = ctas * w;
      best_w = w;
    }
  }
  return best_w;
}

}  // namespace fnb

#define FNB_CUDA_OK(expr)                                   \
  do {                                                      \
    cudaError_t fnb_e_ = (expr);                            \
    if (fnb_e_ != cudaSuccess) return fnb_cuda_fail(fnb_e_, #expr); \
  } while (0)
