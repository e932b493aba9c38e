// distance.cu -- K3: compatibility distance of every genome against S
// species representatives (distance, ops.hpp:415-473), FP64, bit-exact.
//
// The reference walks g1's rows in row order, looks each marker up in g2 by
// linear scan and accumulates the attribute differences sequentially.  Here:
//   * k_union_build merges the S representatives into ONE marker table per
//     gene class: a key maps to a bitmask of the representatives holding it
//     and to a packed run of their attributes (the lowest row's, which is
//     what the reference's first-match find_conn / find_node returns,
//     genome.hpp:195-210).  The tables are 2-choice cuckoo tables with
//     2-slot buckets, so a lookup is two 16-byte loads and no probe loop
//     (no divergence across the warp).  Tables and attribute runs form one
//     image that k_distance copies into shared memory when it fits (a random
//     gather from shared memory costs a few wavefronts; from L1 one per
//     distinct line);
//   * k_distance: one warp per genome, 32 rows per step (one per lane,
//     coalesced, prefetched three steps ahead).  Each lane probes its row
//     once; for every representative s present in the step the lanes write
//     their term (+0.0 when unmatched) into an FP64 tile; a 32x32 bit
//     transpose of the lanes' masks gives lane s the rows matching
//     representative s, and lane s adds its tile row in row order.  Adding
//     +0.0 for an unmatched row is exact (every term is >= +0 and the sums
//     start at +0), so each sum is the reference's g1 row-order sum bit for
//     bit.
#include <algorithm>

#include "distance_warp.cuh"

namespace fnb {

struct __align__(16) NodeEnt {
  double bias, resp, agg, act;
};

struct UnionHdr {
  uint32_t nb_c, nb_n;        // cuckoo buckets (2 slots each)
  uint32_t seed_c, seed_n;
  uint32_t off_ckeys, off_cmeta, off_cw, conn_bytes;    // image sections (bytes from the image start)
  uint32_t off_nkeys, off_nmeta, off_nent, node_bytes;  // node sections (relative to the node part)
  int n_cent, n_nent, u_c, u_n;
  uint32_t off_ncode;         // compact node entries: agg | act << 16 codes
  int bad_codes;              // a representative's agg/act is not a small integer
  int compact;                // 32-bit meta (mask | run << 16) and 16-byte node entries + codes
  int pad;
  int counts[2 * 32];         // [s][node, conn] non-empty rows of representative s
};

// Compact image format: S <= 16, fewer than 2^16 entries per class and every
// representative node's agg / act a small integer.  Node agg / act then
// compare through 16-bit codes: a genome value that is not a small integer
// gets 0xFFFF, which no representative has, so code equality is exactly the
// reference's double comparison (ops.hpp:432-433).
__host__ __device__ __forceinline__ bool small_int(double v) { return v >= 0.0 && v < 32768.0 && v == double(int(v)); }
__device__ __forceinline__ uint32_t attr_code(double v) { return small_int(v) ? uint32_t(int(v)) : 0xFFFFu; }

// ---- hashing -----------------------------------------------------------------
__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x7feb352du;
  h ^= h >> 15;
  h *= 0x846ca68bu;
  h ^= h >> 16;
  return h;
}
__device__ __forceinline__ uint32_t key_mix(unsigned long long k, uint32_t seed) {
  return fmix32(uint32_t(k) * 0x9E3779B1u ^ uint32_t(k >> 32) * 0x85EBCA77u ^ seed);
}
// the two candidate buckets: high bits of the mix, and of a bijective remix of it
__device__ __forceinline__ uint32_t bucket_a(uint32_t h, uint32_t nb) { return __umulhi(h, nb); }
// (never bucket_a: a key always has two distinct buckets)
__device__ __forceinline__ uint32_t bucket_b(uint32_t h, uint32_t nb) {
  const uint32_t g = h * 0xC2B2AE3Du + 0x27D4EB2Fu;
  const uint32_t a = __umulhi(h, nb);
  const uint32_t b = __umulhi(g ^ (g >> 15), nb - 1);  // nb >= 16
  return b >= a ? b + 1 : b;
}
__device__ __forceinline__ uint32_t bucket1(unsigned long long k, uint32_t seed, uint32_t nb) {
  return bucket_a(key_mix(k, seed), nb);
}
__device__ __forceinline__ uint32_t bucket2(unsigned long long k, uint32_t seed, uint32_t nb) {
  return bucket_b(key_mix(k, seed), nb);
}
// dedup tables of the build (power of two, linear probing)
__device__ __forceinline__ uint32_t dhash(unsigned long long k) {
  return fmix32(uint32_t(k) * 0x9E3779B1u ^ uint32_t(k >> 32) * 0x85EBCA77u);
}

struct DSlot {                // dedup slot
  unsigned long long key;
  uint32_t mask;              // representatives holding the key
  uint32_t idx;               // distinct-key index (after compaction)
};

struct UnionView {
  UnionHdr* hdr;
  DSlot *dc, *dn;             // dedup tables
  uint32_t dcap_c, dcap_n;
  unsigned long long *lk_c, *lk_n;  // distinct keys
  uint32_t *lm_c, *lm_n;      // their masks
  uint32_t *lb_c, *lb_n;      // their entry runs
  uint32_t *id_c, *id_n;      // cuckoo slot -> distinct-key index, when the CTA's shared memory is too small
  int *rmin_c, *rmin_n;       // lowest representative row per entry
  uint8_t* img;               // connection part at 0, node part at img_off_node
  size_t img_off_node, img_cap;
  uint32_t smem_cuckoo;       // dynamic shared memory of k_ub_cuckoo
  int sc, sn;                 // S*C, S*N
  int S;
};

__host__ inline uint32_t pow2_at_least(size_t n) {
  uint32_t h = 16;
  while (h < n) h <<= 1;
  return h;
}
__host__ __device__ inline uint32_t align16u(uint32_t x) { return (x + 15u) & ~15u; }

// image bytes for nb buckets and n entries of a class (entry size e)
__host__ __device__ inline uint32_t class_bytes(uint32_t nb, uint32_t n, uint32_t e) {
  return 2u * nb * 8u * 2u + align16u(n * e);
}

constexpr uint32_t kCuckooSmem = 200 * 1024;

// scratch layout; nb <= max(S*C, kCuckooSmem / 8) buckets per class
__host__ inline size_t union_bytes(int S, int N, int C, UnionView* v, void* base) {
  const size_t dcc = pow2_at_least(2 * size_t(S) * C), dcn = pow2_at_least(2 * size_t(S) * N);
  const size_t SC = size_t(S) * C, SN = size_t(S) * N;
  const size_t nbc = std::max(SC, size_t(kCuckooSmem / 8)), nbn = std::max(SN, size_t(kCuckooSmem / 8));
  uint8_t* p = static_cast<uint8_t*>(base);
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += (bytes + 255) & ~size_t(255);
    return r;
  };
  UnionView u;
  u.hdr = reinterpret_cast<UnionHdr*>(take(sizeof(UnionHdr)));
  u.dc = reinterpret_cast<DSlot*>(take(dcc * sizeof(DSlot)));
  u.dn = reinterpret_cast<DSlot*>(take(dcn * sizeof(DSlot)));
  u.lk_c = reinterpret_cast<unsigned long long*>(take(SC * 8));
  u.lk_n = reinterpret_cast<unsigned long long*>(take(SN * 8));
  u.lm_c = reinterpret_cast<uint32_t*>(take(SC * 4));
  u.lm_n = reinterpret_cast<uint32_t*>(take(SN * 4));
  u.lb_c = reinterpret_cast<uint32_t*>(take(SC * 4));
  u.lb_n = reinterpret_cast<uint32_t*>(take(SN * 4));
  u.id_c = reinterpret_cast<uint32_t*>(take(2 * nbc * 4));
  u.id_n = reinterpret_cast<uint32_t*>(take(2 * nbn * 4));
  u.rmin_c = reinterpret_cast<int*>(take(SC * 4));
  u.rmin_n = reinterpret_cast<int*>(take(SN * 4));
  u.img_off_node = (32 * nbc + 8 * SC + 255) & ~size_t(255);
  u.img_cap = u.img_off_node + 32 * nbn + 36 * SN + 64;
  u.img = take(u.img_cap);
  u.dcap_c = uint32_t(dcc);
  u.dcap_n = uint32_t(dcn);
  u.smem_cuckoo = kCuckooSmem;
  u.sc = int(SC);
  u.sn = int(SN);
  u.S = S;
  if (v) *v = u;
  return size_t(p - static_cast<uint8_t*>(base)) + 256;
}

constexpr uint32_t kNoId = 0xffffffffu;

// ---- build: five small grid kernels + one cuckoo CTA per class ----------------
__device__ __forceinline__ uint32_t dedup_insert(DSlot* t, uint32_t cap, unsigned long long key) {
  uint32_t s = dhash(key) & (cap - 1);
  for (;;) {
    const unsigned long long prev = atomicCAS(&t[s].key, kEmptyKey, key);
    if (prev == kEmptyKey || prev == key) return s;
    s = (s + 1) & (cap - 1);
  }
}
__device__ __forceinline__ const DSlot* dedup_find(const DSlot* t, uint32_t cap, unsigned long long key) {
  uint32_t s = dhash(key) & (cap - 1);
  while (t[s].key != key) s = (s + 1) & (cap - 1);
  return &t[s];
}

__global__ void k_ub_clear(UnionView u, int S, int N, int C) {
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x, n = gridDim.x * blockDim.x;
  for (uint32_t i = i0; i < u.dcap_c; i += n) u.dc[i] = DSlot{kEmptyKey, 0u, 0u};
  for (uint32_t i = i0; i < u.dcap_n; i += n) u.dn[i] = DSlot{kEmptyKey, 0u, 0u};
  for (int i = i0; i < S * C; i += n) u.rmin_c[i] = 0x7fffffff;
  for (int i = i0; i < S * N; i += n) u.rmin_n[i] = 0x7fffffff;
  if (i0 < 64) u.hdr->counts[i0] = 0;
  if (i0 == 0) u.hdr->n_cent = u.hdr->n_nent = u.hdr->u_c = u.hdr->u_n = u.hdr->bad_codes = 0;
}

// 1. distinct keys, the representatives holding them, non-empty row counts
__global__ void k_ub_insert(const double* __restrict__ rn, const double* __restrict__ rc, int S, int N, int C,
                            UnionView u) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < S * C) {
    const int s = i / C;
    const double* row = rc + size_t(i) * kConnCols;
    if (isnan(row[kIn])) return;
    atomicOr(&u.dc[dedup_insert(u.dc, u.dcap_c, conn_key(row[kIn], row[kOut]))].mask, 1u << s);
    atomicAdd(&u.hdr->counts[2 * s + 1], 1);
  } else if (i < S * C + S * N) {
    const int k = i - S * C, s = k / N;
    const double key = rn[size_t(k) * kNodeCols + kKey];
    if (isnan(key)) return;
    atomicOr(&u.dn[dedup_insert(u.dn, u.dcap_n, node_key(key))].mask, 1u << s);
    atomicAdd(&u.hdr->counts[2 * s], 1);
    const double* row = rn + size_t(k) * kNodeCols;
    if (!small_int(row[kAgg]) || !small_int(row[kAct])) u.hdr->bad_codes = 1;
  }
}

__device__ __forceinline__ bool use_compact(const UnionView& u) {
  const UnionHdr* h = u.hdr;
  return u.S <= 16 && h->n_cent < 65536 && h->n_nent < 65536 && !h->bad_codes;
}

// 2. distinct-key lists and their packed entry runs
__global__ void k_ub_compact(UnionView u) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < u.dcap_c) {
    const DSlot q = u.dc[i];
    if (q.key == kEmptyKey) return;
    const int j = atomicAdd(&u.hdr->u_c, 1);
    u.dc[i].idx = uint32_t(j);
    u.lk_c[j] = q.key;
    u.lm_c[j] = q.mask;
    u.lb_c[j] = uint32_t(atomicAdd(&u.hdr->n_cent, __popc(q.mask)));
  } else if (i < u.dcap_c + u.dcap_n) {
    const uint32_t k = i - u.dcap_c;
    const DSlot q = u.dn[k];
    if (q.key == kEmptyKey) return;
    const int j = atomicAdd(&u.hdr->u_n, 1);
    u.dn[k].idx = uint32_t(j);
    u.lk_n[j] = q.key;
    u.lm_n[j] = q.mask;
    u.lb_n[j] = uint32_t(atomicAdd(&u.hdr->n_nent, __popc(q.mask)));
  }
}

// 3. lowest row of representative s per key (entry = run + rank of s in the mask)
__global__ void k_ub_rmin(const double* __restrict__ rn, const double* __restrict__ rc, int S, int N, int C,
                          UnionView u) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < S * C) {
    const int s = i / C;
    const double* row = rc + size_t(i) * kConnCols;
    if (isnan(row[kIn])) return;
    const uint32_t j = dedup_find(u.dc, u.dcap_c, conn_key(row[kIn], row[kOut]))->idx;
    atomicMin(&u.rmin_c[u.lb_c[j] + __popc(u.lm_c[j] & ((1u << s) - 1u))], i);
  } else if (i < S * C + S * N) {
    const int k = i - S * C, s = k / N;
    const double key = rn[size_t(k) * kNodeCols + kKey];
    if (isnan(key)) return;
    const uint32_t j = dedup_find(u.dn, u.dcap_n, node_key(key))->idx;
    atomicMin(&u.rmin_n[u.lb_n[j] + __popc(u.lm_n[j] & ((1u << s) - 1u))], k);
  }
}

// 5. attribute entries (connection weights / node attributes of those rows)
//    right after each class's cuckoo sections; finalises the image header
__global__ void k_ub_fill(const double* __restrict__ rn, const double* __restrict__ rc, UnionView u) {
  UnionHdr* h = u.hdr;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int ec = h->n_cent, en = h->n_nent;
  const bool compact = use_compact(u);
  const uint32_t meta = compact ? 4u : 8u;  // bytes per slot
  const uint32_t off_cw = align16u((16u + 2u * meta) * h->nb_c), off_nent = align16u((16u + 2u * meta) * h->nb_n);
  const uint32_t off_ncode = off_nent + uint32_t(en) * (compact ? 16u : 32u);
  uint8_t* nimg = u.img + u.img_off_node;
  if (i < ec) {
    reinterpret_cast<double*>(u.img + off_cw)[i] = rc[size_t(u.rmin_c[i]) * kConnCols + kW];
  } else if (i < ec + en) {
    const int e = i - ec;
    const double* b = rn + size_t(u.rmin_n[e]) * kNodeCols;
    if (compact) {
      reinterpret_cast<double2*>(nimg + off_nent)[e] = make_double2(b[kBias], b[kResp]);
      reinterpret_cast<uint32_t*>(nimg + off_ncode)[e] = attr_code(b[kAgg]) | (attr_code(b[kAct]) << 16);
    } else {
      reinterpret_cast<NodeEnt*>(nimg + off_nent)[e] = NodeEnt{b[kBias], b[kResp], b[kAgg], b[kAct]};
    }
  }
  if (i == 0) {
    h->compact = compact ? 1 : 0;
    h->off_cw = off_cw;
    h->conn_bytes = off_cw + align16u(uint32_t(ec) * 8u);
    h->off_nent = off_nent;
    h->off_ncode = off_ncode;
    h->node_bytes = compact ? off_ncode + align16u(uint32_t(en) * 4u) : off_ncode;
  }
}

// Lock-free parallel cuckoo placement of distinct keys [0, U) into 2*nb
// shared-memory slots (Alcantara-style: every thread holds one key; a full
// bucket evicts a pseudo-randomly chosen slot with atomicExch and the victim
// moves to its other bucket).  Returns false on a too-long chain.
__device__ bool cuckoo_place(uint32_t* ids, const unsigned long long* keys, int U, uint32_t nb, uint32_t seed) {
  bool ok = true;
  for (int i = threadIdx.x; i < U; i += blockDim.x) {
    uint32_t cur = uint32_t(i);
    uint32_t b = bucket1(keys[cur], seed, nb);
    bool placed = false;
    const int max_it = min(1024, 16 * U + 64);  // a placeable key rarely needs more evictions
    for (int it = 0; it < max_it && !placed; ++it) {
      for (int j = 0; j < 2 && !placed; ++j) placed = atomicCAS(&ids[2 * b + j], kNoId, cur) == kNoId;
      if (!placed && it == 0) {  // a fresh key also tries its second bucket before evicting
        const uint32_t b2 = bucket2(keys[cur], seed, nb);
        for (int j = 0; j < 2 && !placed; ++j) placed = atomicCAS(&ids[2 * b2 + j], kNoId, cur) == kNoId;
      }
      if (placed) break;
      cur = atomicExch(&ids[2 * b + (fmix32(cur * 0x9E3779B1u + uint32_t(it)) & 1u)], cur);
      const unsigned long long vk = keys[cur];
      const uint32_t v1 = bucket1(vk, seed, nb);
      b = b == v1 ? bucket2(vk, seed, nb) : v1;
    }
    ok = ok && placed;
  }
  return ok;
}

// 4. cuckoo tables, one CTA per class (0: connections, 1: nodes), placed
//    in shared memory when it holds them (else in the global id buffer); a
//    failed placement is redone with a new seed and, every fourth try, 1/8
//    more buckets.  Writes the class's key and meta sections of the image.
__global__ void __launch_bounds__(1024) k_ub_cuckoo(UnionView u) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int s_fail;
  const bool conn = blockIdx.x == 0;
  const int U = conn ? u.hdr->u_c : u.hdr->u_n;
  const unsigned long long* lk = conn ? u.lk_c : u.lk_n;
  const uint32_t* lm = conn ? u.lm_c : u.lm_n;
  const uint32_t* lb = conn ? u.lb_c : u.lb_n;
  const uint32_t key_bytes = align16u(uint32_t(U) * 8u);
  uint32_t nb = max(16u, uint32_t((U * 10 + 13) / 14));  // load <= 0.7
  // keys in shared memory if they leave room for twice the first table
  const bool keys_sm = key_bytes + 16u * nb <= u.smem_cuckoo;
  const uint32_t room = u.smem_cuckoo - (keys_sm ? key_bytes : 0u);
  const bool ids_sm = 8u * nb <= room;
  const unsigned long long* keys = lk;
  if (keys_sm) {
    unsigned long long* k = reinterpret_cast<unsigned long long*>(sm);
    for (int i = threadIdx.x; i < U; i += blockDim.x) k[i] = lk[i];
    keys = k;
  }
  uint32_t* ids = ids_sm ? reinterpret_cast<uint32_t*>(sm + (keys_sm ? key_bytes : 0u)) : (conn ? u.id_c : u.id_n);
  const uint32_t max_nb = ids_sm ? room / 8u : uint32_t(max(conn ? u.sc : u.sn, int(kCuckooSmem / 8)));
  uint32_t seed = 0;
  for (int attempt = 0;; ++attempt) {
    if (attempt > 0 && attempt % 4 == 0) nb = min(max_nb, nb + nb / 8 + 1);
    seed = 0x51ED2701u + uint32_t(attempt) * 0x9E3779B9u;
    for (uint32_t i = threadIdx.x; i < 2 * nb; i += blockDim.x) ids[i] = kNoId;
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    if (!cuckoo_place(ids, keys, U, nb, seed)) s_fail = 1;
    __syncthreads();
    if (!s_fail) break;
    __syncthreads();
  }
  uint8_t* img = u.img + (conn ? 0 : u.img_off_node);
  unsigned long long* tk = reinterpret_cast<unsigned long long*>(img);
  const bool compact = use_compact(u);
  for (uint32_t i = threadIdx.x; i < 2 * nb; i += blockDim.x) {
    const uint32_t id = ids[i];
    tk[i] = id == kNoId ? kEmptyKey : keys[id];
    if (compact)
      reinterpret_cast<uint32_t*>(tk + 2 * nb)[i] = id == kNoId ? 0u : (lm[id] | (lb[id] << 16));
    else
      (tk + 2 * nb)[i] = id == kNoId ? 0ull : (lm[id] | (static_cast<unsigned long long>(lb[id]) << 32));
  }
  if (threadIdx.x == 0) {
    UnionHdr* h = u.hdr;
    if (conn) {
      h->nb_c = nb;
      h->seed_c = seed;
      h->off_ckeys = 0;
      h->off_cmeta = 16u * nb;
    } else {
      h->nb_n = nb;
      h->seed_n = seed;
      h->off_nkeys = 0;
      h->off_nmeta = 16u * nb;
    }
  }
}

// ---- distance kernel ------------------------------------------------------------
constexpr unsigned kFull = 0xffffffffu;
constexpr int kDistWarps = 20;  // one 640-thread CTA per SM
constexpr int kTileStride = 34;  // doubles per tile row (16-byte rows, conflict-light LDS.128)

struct ClassTab {
  const unsigned long long* keys;  // 2 * nb slots
  const void* meta;                // per slot: mask | run << 32 (u64), or mask | run << 16 (u32, compact)
  const void* ent;                 // attribute runs
  const uint32_t* codes;           // compact node entries: agg | act << 16
  uint32_t nb, seed;
};

// (mask, run) of `key`; mask 0 if absent.  Two 16-byte bucket loads, no loop.
template <bool kCompact>
__device__ __forceinline__ void cuckoo_lookup(const ClassTab& t, unsigned long long key, uint32_t& msk,
                                              uint32_t& run) {
  const uint32_t h = key_mix(key, t.seed);
  const uint32_t b1 = bucket_a(h, t.nb), b2 = bucket_b(h, t.nb);
  const ulonglong2 k1 = reinterpret_cast<const ulonglong2*>(t.keys)[b1];
  const ulonglong2 k2 = reinterpret_cast<const ulonglong2*>(t.keys)[b2];
  int slot = -1;
  slot = k2.y == key ? int(2 * b2 + 1) : slot;
  slot = k2.x == key ? int(2 * b2) : slot;
  slot = k1.y == key ? int(2 * b1 + 1) : slot;
  slot = k1.x == key ? int(2 * b1) : slot;
  msk = 0u;
  run = 0u;
  if (slot >= 0) {
    if (kCompact) {
      const uint32_t m = static_cast<const uint32_t*>(t.meta)[slot];
      msk = m & 0xFFFFu;
      run = m >> 16;
    } else {
      const unsigned long long m = static_cast<const unsigned long long*>(t.meta)[slot];
      msk = uint32_t(m);
      run = uint32_t(m >> 32);
    }
  }
}

// 32x32 bit transpose across the warp: returns, for lane s, the mask of lanes
// whose `x` has bit s set (five butterfly rounds of shfl_xor).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int j = 16, i = 0; j >= 1; j >>= 1, ++i) {
    const uint32_t m = j == 16 ? 0x0000ffffu : j == 8 ? 0x00ff00ffu : j == 4 ? 0x0f0f0f0fu : j == 2 ? 0x33333333u
                                                                                                     : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(kFull, x, j);
    x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

// lane s adds its tile row (the step's terms for representative s) in row order
__device__ __forceinline__ void add_tile_row(const double* row, uint32_t my, bool dense, double& sum) {
  if (dense) {  // every entry (+0.0 where unmatched)
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const double2 v = *reinterpret_cast<const double2*>(row + i);
      sum = __dadd_rn(sum, v.x);
      sum = __dadd_rn(sum, v.y);
    }
  } else {
    for (; my & (my - 1u); my &= my - 1u, my &= my - 1u) {  // two per step, loads issued together
      const double v0 = row[__ffs(my) - 1];
      const double v1 = row[__ffs(my & (my - 1u)) - 1];
      sum = __dadd_rn(sum, v0);
      sum = __dadd_rn(sum, v1);
    }
    if (my) sum = __dadd_rn(sum, row[__ffs(my) - 1]);
  }
}

struct DistArgs {
  const double* nodes;
  const double* conns;
  int P, S, N, C;
  double cd, ch;
  double* out;
  const int* only_unassigned;
  const int* after_founder;
};

// ops.hpp:443-470: one gene class's contribution
__device__ __forceinline__ double class_term(double total, int n1, int n2, int m, double sum, double cd, double ch) {
  const int disjoint = (n1 - m) + (n2 - m);
  const int norm = max(1, max(n1, n2));
  total = __dadd_rn(total, __ddiv_rn(__dmul_rn(cd, double(disjoint)), double(norm)));
  if (m > 0) total = __dadd_rn(total, __ddiv_rn(__dmul_rn(ch, sum), double(m)));
  return total;
}

struct ConnRow {
  double2 io;  // in, out
  double w;
};
struct NodeRow {
  double k, b, r, ag, ac;
};

// The warp's genomes as one stream of 32-row steps: the cursor walks the
// conn (or node) steps of successive genomes, skipping masked genomes, so
// the prefetch runs across genome boundaries.
struct Cursor {
  int g, j;         // genome (>= P: exhausted), step inside it
  const double* p;  // this lane's row of step j of genome g
};

__device__ __forceinline__ bool skip_genome(const DistArgs& a, int g) {
  // speciation rounds only need genomes still without a species (and, for a
  // founding round, after the founder): the rest are never read
  if (a.only_unassigned && a.only_unassigned[g] >= 0) return true;
  if (a.after_founder && (a.after_founder[0] < 0 || g <= a.after_founder[0])) return true;
  return false;
}
template <bool kMasked>
__device__ __forceinline__ int valid_from(const DistArgs& a, int g, int stride) {
  if (kMasked)
    while (g < a.P && skip_genome(a, g)) g += stride;
  return g;
}
// Cursor over one gene class: `rows` rows of `cols` doubles per genome; the
// lane's row pointer moves by one 32-row step, or to the next genome
__device__ __forceinline__ Cursor cursor_at(int g, const double* base, int rows, int cols, int lane) {
  return Cursor{g, 0, base + (size_t(g) * rows + lane) * cols};
}
template <bool kMasked>
__device__ __forceinline__ void advance(const DistArgs& a, Cursor& c, int steps, int stride, const double* base,
                                        int rows, int cols, int lane) {
  if (++c.j == steps)
    c = cursor_at(valid_from<kMasked>(a, c.g + stride, stride), base, rows, cols, lane);
  else
    c.p += 32 * cols;
}

__device__ __forceinline__ ConnRow load_conn(const DistArgs& a, const Cursor& c, int lane) {
  ConnRow x;
  x.io = make_double2(__longlong_as_double(0x7ff8000000000000ll), 0.0);
  x.w = 0.0;
  if (c.g < a.P && c.j * 32 + lane < a.C) {
    x.io = __ldg(reinterpret_cast<const double2*>(c.p));
    x.w = __ldg(c.p + kW);
  }
  return x;
}
__device__ __forceinline__ NodeRow load_node(const DistArgs& a, const Cursor& c, int lane) {
  NodeRow x{__longlong_as_double(0x7ff8000000000000ll), 0.0, 0.0, 0.0, 0.0};
  if (c.g < a.P && c.j * 32 + lane < a.N) {
    x.k = __ldg(c.p + kKey);
    x.b = __ldg(c.p + kBias);
    x.r = __ldg(c.p + kResp);
    x.ag = __ldg(c.p + kAgg);
    x.ac = __ldg(c.p + kAct);
  }
  return x;
}

constexpr unsigned kDenseRows = 12;  // a representative matching more rows of a step: add its whole tile row

// One 32-row step after the lookups.  `term(s, e)` is the lane's term
// against representative s from attribute entry e.  A 32x32 bit transpose
// of the lanes' masks gives lane s the rows matching representative s.
// Dense steps write every (s, lane) of the representatives present (+0.0
// where unmatched) and lane s adds its whole tile row; sparse steps write
// only the matches and lane s adds just those, in row order.
template <class Term>
__device__ __forceinline__ void step_terms(uint32_t msk, uint32_t e, int lane, int S, double* tile, int& matched,
                                           double& sum, Term term) {
  const uint32_t wm = __reduce_or_sync(kFull, msk);
  if (!wm) return;
  const uint32_t my = warp_transpose32(msk, lane);
  // representatives matching many rows of the step take their whole tile row
  // (every entry written, +0.0 where unmatched); the others only their matches
  const uint32_t dm = __ballot_sync(kFull, lane < S && uint32_t(__popc(my)) > kDenseRows);
  const bool dense = (dm >> lane) & 1u;
  double* col = tile + lane;
  if (dm) {
    for (uint32_t m = msk | dm; m; m &= m - 1u) {
      const int s = __ffs(m) - 1;
      double t = 0.0;
      if ((msk >> s) & 1u) t = term(s, e++);
      col[s * kTileStride] = t;
    }
  } else {
    for (uint32_t m = msk; m; m &= m - 1u) {
      const int s = __ffs(m) - 1;
      col[s * kTileStride] = term(s, e++);
    }
  }
  __syncwarp();
  if (lane < S) {
    matched += __popc(my);
    if (my) add_tile_row(tile + lane * kTileStride, my, dense, sum);
  }
  __syncwarp();
}

// The per-genome loop.  ClassTab pointers are derived from the shared-memory
// image in the caller's branch, so the compiler emits shared-space loads there.
// A genome's node steps are spread between its connection steps, so the
// one-step node prefetch gets several connection steps of lead time.
template <bool kCompact, bool kMasked>
__device__ __forceinline__ void distance_genomes(const DistArgs& a, const ClassTab& tc, const ClassTab& tn, int n2,
                                                 int c2, double* tile) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.S;
  const int NS = (a.N + 31) / 32, CS = (a.C + 31) / 32;
  const int stride = gridDim.x * kDistWarps;
  const double* cw = static_cast<const double*>(tc.ent);
  const NodeEnt* ne = static_cast<const NodeEnt*>(tn.ent);
  const int g0 = valid_from<kMasked>(a, blockIdx.x * kDistWarps + warp, stride);
  // prefetch: node rows one node step ahead, connection rows three steps ahead
  Cursor nc = cursor_at(g0, a.nodes, a.N, kNodeCols, lane);
  Cursor cc = cursor_at(g0, a.conns, a.C, kConnCols, lane);
  auto next_n = [&]() { advance<kMasked>(a, nc, NS, stride, a.nodes, a.N, kNodeCols, lane); };
  auto next_c = [&]() { advance<kMasked>(a, cc, CS, stride, a.conns, a.C, kConnCols, lane); };
  NodeRow nq = load_node(a, nc, lane);
  next_n();
  ConnRow q0 = load_conn(a, cc, lane);
  next_c();
  ConnRow q1 = load_conn(a, cc, lane);
  next_c();
  ConnRow q2 = load_conn(a, cc, lane);
  next_c();
  for (int g = g0; g < a.P; g = valid_from<kMasked>(a, g + stride, stride)) {
    int n1 = 0, c1 = 0, mn = 0, mc = 0;
    double sum_n = 0.0, sum_c = 0.0;
    int ni = 0;  // next node step
    for (int j = 0; j < CS; ++j) {
      // ---- connection genes: |dw| / 1 (ops.hpp:454-463)
      {
        const ConnRow x = q0;
        q0 = q1;
        q1 = q2;
        q2 = load_conn(a, cc, lane);
        next_c();
        const bool nonempty = !isnan(x.io.x);
        c1 += __popc(__ballot_sync(kFull, nonempty));
        uint32_t msk = 0u, e = 0u;
        if (nonempty) cuckoo_lookup<kCompact>(tc, conn_key(x.io.x, x.io.y), msk, e);
        step_terms(msk, e, lane, S, tile, mc, sum_c,
                   [&](int, uint32_t i) { return fabs(__dsub_rn(x.w, cw[i])); });  // |dw| / 1.0 == |dw|
      }
      // ---- node genes: (|db| + |dr| + [agg!=] + [act!=]) / 4 (ops.hpp:428-441);
      //      spread between the connection steps, the last one takes any left (N > C)
      while (ni < NS && (ni * CS <= j * NS || j == CS - 1)) {
        ++ni;
        const NodeRow x = nq;
        nq = load_node(a, nc, lane);
        next_n();
        const bool nonempty = !isnan(x.k);
        n1 += __popc(__ballot_sync(kFull, nonempty));
        uint32_t msk = 0u, e = 0u;
        if (nonempty) cuckoo_lookup<kCompact>(tn, node_key(x.k), msk, e);
        if (kCompact) {
          const uint32_t code = attr_code(x.ag) | (attr_code(x.ac) << 16);
          const double2* ne2 = static_cast<const double2*>(tn.ent);
          step_terms(msk, e, lane, S, tile, mn, sum_n, [&](int, uint32_t i) {
            const double2 o = ne2[i];
            const uint32_t diff = code ^ tn.codes[i];
            double d = __dadd_rn(fabs(__dsub_rn(x.b, o.x)), fabs(__dsub_rn(x.r, o.y)));
            d = __dadd_rn(d, (diff & 0xFFFFu) ? 1.0 : 0.0);
            d = __dadd_rn(d, (diff >> 16) ? 1.0 : 0.0);
            return __dmul_rn(d, 0.25);  // d * 0.25 == d / 4.0 exactly
          });
        } else {
          step_terms(msk, e, lane, S, tile, mn, sum_n, [&](int, uint32_t i) {
            const NodeEnt o = ne[i];
            double d = __dadd_rn(fabs(__dsub_rn(x.b, o.bias)), fabs(__dsub_rn(x.r, o.resp)));
            d = __dadd_rn(d, x.ag != o.agg ? 1.0 : 0.0);
            d = __dadd_rn(d, x.ac != o.act ? 1.0 : 0.0);
            return __dmul_rn(d, 0.25);  // d * 0.25 == d / 4.0 exactly
          });
        }
      }
    }
    if (lane < S) {
      double total = class_term(0.0, n1, n2, mn, sum_n, a.cd, a.ch);
      total = class_term(total, c1, c2, mc, sum_c, a.cd, a.ch);
      a.out[size_t(g) * S + lane] = total;
    }
  }
}

__device__ __forceinline__ void copy16(uint8_t* dst, const uint8_t* src, uint32_t bytes) {
  for (uint32_t i = threadIdx.x; i < bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
}

__device__ __forceinline__ ClassTab conn_tab(const uint8_t* img, const UnionHdr* h) {
  return ClassTab{reinterpret_cast<const unsigned long long*>(img + h->off_ckeys), img + h->off_cmeta,
                  img + h->off_cw, nullptr, h->nb_c, h->seed_c};
}
__device__ __forceinline__ ClassTab node_tab(const uint8_t* img, const UnionHdr* h) {
  return ClassTab{reinterpret_cast<const unsigned long long*>(img + h->off_nkeys), img + h->off_nmeta,
                  img + h->off_nent, reinterpret_cast<const uint32_t*>(img + h->off_ncode), h->nb_n, h->seed_n};
}

template <bool kCompact, bool kMasked>
__device__ __forceinline__ void distance_placed(const DistArgs& a, const UnionView& u, uint32_t smem_img_cap,
                                                double* tile, uint8_t* simg, int n2, int c2) {
  const UnionHdr* h = u.hdr;
  const uint32_t cb = h->conn_bytes, nbytes = h->node_bytes;
  const uint8_t* gnode = u.img + u.img_off_node;
  // CTA-uniform placement: the connection image first (it carries the hot
  // lookups), the node image after it if it still fits
  if (cb + nbytes <= smem_img_cap) {
    copy16(simg, u.img, cb);
    copy16(simg + cb, gnode, align16u(nbytes));
    __syncthreads();
    distance_genomes<kCompact, kMasked>(a, conn_tab(simg, h), node_tab(simg + cb, h), n2, c2, tile);
  } else if (cb <= smem_img_cap) {
    copy16(simg, u.img, cb);
    __syncthreads();
    distance_genomes<kCompact, kMasked>(a, conn_tab(simg, h), node_tab(gnode, h), n2, c2, tile);
  } else {
    distance_genomes<kCompact, kMasked>(a, conn_tab(u.img, h), node_tab(gnode, h), n2, c2, tile);
  }
}

// persistent: one 512-thread CTA per SM, one warp per genome
__global__ void __launch_bounds__(kDistWarps * 32, 1)
k_distance(DistArgs a, UnionView u, uint32_t smem_img_cap) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* tile = reinterpret_cast<double*>(smem_raw) + size_t(warp) * a.S * kTileStride;
  uint8_t* simg = smem_raw + size_t(kDistWarps) * a.S * kTileStride * sizeof(double);
  const UnionHdr* h = u.hdr;
  const int n2 = lane < a.S ? h->counts[2 * lane] : 0, c2 = lane < a.S ? h->counts[2 * lane + 1] : 0;
  const bool masked = a.only_unassigned != nullptr || a.after_founder != nullptr;
  if (h->compact) {
    if (masked) distance_placed<true, true>(a, u, smem_img_cap, tile, simg, n2, c2);
    else distance_placed<true, false>(a, u, smem_img_cap, tile, simg, n2, c2);
  } else {
    if (masked) distance_placed<false, true>(a, u, smem_img_cap, tile, simg, n2, c2);
    else distance_placed<false, false>(a, u, smem_img_cap, tile, simg, n2, c2);
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
  if (S > 32) return cudaErrorInvalidValue;
  UnionView u;
  if (union_bytes(S, N, C, &u, scratch) > scratch_bytes) return cudaErrorInvalidValue;
  const int rows = S * (C + N);
  k_ub_clear<<<64, 256, 0, st>>>(u, S, N, C);
  k_ub_insert<<<(rows + 255) / 256, 256, 0, st>>>(rn, rc, S, N, C, u);
  k_ub_compact<<<int((size_t(u.dcap_c) + u.dcap_n + 255) / 256), 256, 0, st>>>(u);
  k_ub_rmin<<<(rows + 255) / 256, 256, 0, st>>>(rn, rc, S, N, C, u);
  cudaError_t e = cudaFuncSetAttribute(k_ub_cuckoo, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCuckooSmem));
  if (e != cudaSuccess) return e;
  k_ub_cuckoo<<<2, 1024, kCuckooSmem, st>>>(u);
  k_ub_fill<<<(rows + 255) / 256, 256, 0, st>>>(rn, rc, u);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // tiles + room for the image's upper bound, capped by the opt-in limit; the
  // kernel reads the real image size and keeps what does not fit in global memory
  const size_t tiles = size_t(kDistWarps) * S * kTileStride * sizeof(double);
  const size_t room = optin > int(tiles) + 1024 ? (size_t(optin) - tiles - 1024) & ~size_t(15) : 0;
  const size_t cap = std::min(u.img_cap, room);  // >= conn + node bytes of any image that fits
  const size_t smem = tiles + cap;
  e = cudaFuncSetAttribute(k_distance, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  const int grid = std::max(1, std::min((P + kDistWarps - 1) / kDistWarps, sms));
  DistArgs a{nodes, conns, P, S, N, C, cd, ch, out, only_unassigned, after_founder};
  k_distance<<<grid, kDistWarps * 32, smem, st>>>(a, u, uint32_t(cap));
  return cudaGetLastError();
}

size_t distance_scratch_bytes(int S, int N, int C) { return union_bytes(S, N, C, nullptr, nullptr); }

}  // namespace fnb
