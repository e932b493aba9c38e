// validate.cu -- explain_invalid (genome.hpp:364-417) as a population-wide
// device validator: one warp per genome, the reference's checks in the
// reference's order, so the first failing check (and its row / key) is the
// one the reference would report:
//   node rows in row order: partially NaN, non-integral or negative key,
//   bad aggregation id, bad activation id; then duplicate node key; input
//   keys, output keys (in their list order); connection rows in row order:
//   partially NaN, non-boolean enabled flag, non-integral or negative
//   endpoint, reference to a missing node; then duplicate connection pair.
// Keys and pairs go into per-warp shared-memory marker tables, so the
// reference's sort + adjacent_find / binary_search become ~1 probe each.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <string>

#include "ctx_internal.cuh"
#include "keytable.cuh"

namespace fnb {

enum ValidCode : int32_t {
  kValid = 0,
  kNodePartial = 1,   // detail = row
  kNodeKey = 2,       // detail = row
  kNodeAgg = 3,       // detail = row
  kNodeAct = 4,       // detail = row
  kDupKey = 5,
  kInputMissing = 6,  // detail = key
  kOutputMissing = 7, // detail = key
  kConnPartial = 8,   // detail = row
  kConnEnabled = 9,   // detail = row
  kConnEndpoint = 10, // detail = row
  kConnMissing = 11,  // detail = row
  kDupPair = 12,
};

__device__ __forceinline__ bool integral(double v) { return v == floor(v); }
// int(v) as the reference's x86-64 build computes it (cvttsd2si): values
// outside the int range, and NaN, become INT_MIN
__device__ __forceinline__ int x86_int(double v) {
  return (v > -2147483649.0 && v < 2147483648.0) ? int(v) : INT_MIN;
}
__device__ __forceinline__ bool key_in(const unsigned long long* t, uint32_t mask, unsigned long long key) {
  uint32_t s = hash_key(key) & mask;
  for (;;) {
    if (t[s] == key) return true;
    if (t[s] == kEmptyKey) return false;
    s = (s + 1) & mask;
  }
}
// insert; true if the key was already present
__device__ __forceinline__ bool key_insert(unsigned long long* t, uint32_t mask, unsigned long long key) {
  uint32_t s = hash_key(key) & mask;
  for (;;) {
    const unsigned long long prev = atomicCAS(&t[s], kEmptyKey, key);
    if (prev == kEmptyKey) return false;
    if (prev == key) return true;
    s = (s + 1) & mask;
  }
}

// first lane (row order) with a failure, as (code, row); code 0 = none
__device__ __forceinline__ void first_fail(int code, int row, int& out_code, int& out_row) {
  const unsigned m = __ballot_sync(0xffffffffu, code != 0);
  if (m && out_code == 0) {
    const int l = __ffs(m) - 1;
    out_code = __shfl_sync(0xffffffffu, code, l);
    out_row = __shfl_sync(0xffffffffu, row, l);
  }
}

__global__ void __launch_bounds__(128)
k_validate(const double* __restrict__ nodes, const double* __restrict__ conns, int P, DevShape sh,
           int32_t* __restrict__ code_out, int32_t* __restrict__ detail_out, size_t smem_per_warp) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x * (blockDim.x >> 5) + warp;
  if (g >= P) return;
  const int N = sh.N, C = sh.C;
  const int Hn = table_capacity(N), Hc = table_capacity(C);
  uint8_t* base = smem_raw + size_t(warp) * smem_per_warp;
  unsigned long long* nk = reinterpret_cast<unsigned long long*>(base);  // node keys (uint32)
  unsigned long long* ck = nk + Hn;                                       // connection pairs
  const double* n = nodes + size_t(g) * N * kNodeCols;
  const double* c = conns + size_t(g) * C * kConnCols;
  for (int i = lane; i < Hn; i += 32) nk[i] = kEmptyKey;
  for (int i = lane; i < Hc; i += 32) ck[i] = kEmptyKey;
  __syncwarp();
  int code = 0, detail = 0;
  bool dup = false;
  // ---- node rows
  for (int r0 = 0; r0 < N && code == 0; r0 += 32) {
    const int r = r0 + lane;
    int my = 0;
    if (r < N) {
      const double* row = n + r * kNodeCols;
      bool all_nan = true, all_fin = true;
#pragma unroll
      for (int a = 0; a < kNodeCols; ++a) {
        all_nan = all_nan && isnan(row[a]);
        all_fin = all_fin && isfinite(row[a]);
      }
      if (!all_nan) {
        const double key = row[kKey], ag = row[kAgg], ac = row[kAct];
        if (!all_fin) my = kNodePartial;
        else if (key < 0 || !integral(key)) my = kNodeKey;
        else if (!integral(ag) || x86_int(ag) < 0 || x86_int(ag) >= sh.n_agg) my = kNodeAgg;
        else if (!integral(ac) || x86_int(ac) < 0 || x86_int(ac) >= sh.n_act) my = kNodeAct;
        else if (key_insert(nk, uint32_t(Hn - 1), uint32_t(x86_int(key)))) dup = true;  // a second row with the key
      }
    }
    first_fail(my, r, code, detail);
  }
  __syncwarp();
  if (code == 0 && __any_sync(0xffffffffu, dup)) code = kDupKey;
  auto has_key = [&](int k) { return key_in(nk, uint32_t(Hn - 1), uint32_t(k)); };
  // ---- required inputs, then outputs (list order)
  if (code == 0) {
    for (int i0 = 0; i0 < sh.I && code == 0; i0 += 32) {
      const int i = i0 + lane;
      const int miss = (i < sh.I && !has_key(sh.input_keys[i])) ? kInputMissing : 0;
      first_fail(miss, i < sh.I ? sh.input_keys[i] : 0, code, detail);
    }
    for (int i0 = 0; i0 < sh.O && code == 0; i0 += 32) {
      const int i = i0 + lane;
      const int miss = (i < sh.O && !has_key(sh.output_keys[i])) ? kOutputMissing : 0;
      first_fail(miss, i < sh.O ? sh.output_keys[i] : 0, code, detail);
    }
  }
  // ---- connection rows
  dup = false;
  for (int r0 = 0; r0 < C && code == 0; r0 += 32) {
    const int r = r0 + lane;
    int my = 0;
    if (r < C) {
      const double* row = c + r * kConnCols;
      bool all_nan = true, all_fin = true;
#pragma unroll
      for (int a = 0; a < kConnCols; ++a) {
        all_nan = all_nan && isnan(row[a]);
        all_fin = all_fin && isfinite(row[a]);
      }
      if (!all_nan) {
        const double in = row[kIn], out = row[kOut], e = row[kEn];
        if (!all_fin) my = kConnPartial;
        else if (e != 0.0 && e != 1.0) my = kConnEnabled;
        else if (!integral(in) || !integral(out) || x86_int(in) < 0 || x86_int(out) < 0) my = kConnEndpoint;
        else if (!has_key(x86_int(in)) || !has_key(x86_int(out))) my = kConnMissing;
        else if (key_insert(ck, uint32_t(Hc - 1),
                            (static_cast<unsigned long long>(uint32_t(x86_int(in))) << 32) | uint32_t(x86_int(out))))
          dup = true;
      }
    }
    first_fail(my, r, code, detail);
  }
  if (code == 0 && __any_sync(0xffffffffu, dup)) code = kDupPair;
  if (lane == 0) {
    code_out[g] = code;
    detail_out[g] = detail;
  }
}

std::string validate_message(int code, int detail) {
  char buf[96];
  switch (code) {
    case kNodePartial: std::snprintf(buf, sizeof buf, "node row %d partially NaN", detail); break;
    case kNodeKey: std::snprintf(buf, sizeof buf, "node row %d has non-integral key", detail); break;
    case kNodeAgg: std::snprintf(buf, sizeof buf, "node row %d has bad aggregation id", detail); break;
    case kNodeAct: std::snprintf(buf, sizeof buf, "node row %d has bad activation id", detail); break;
    case kDupKey: return "duplicate node key";
    case kInputMissing: std::snprintf(buf, sizeof buf, "input key %d missing", detail); break;
    case kOutputMissing: std::snprintf(buf, sizeof buf, "output key %d missing", detail); break;
    case kConnPartial: std::snprintf(buf, sizeof buf, "conn row %d partially NaN", detail); break;
    case kConnEnabled: std::snprintf(buf, sizeof buf, "conn row %d has non-boolean enabled flag", detail); break;
    case kConnEndpoint: std::snprintf(buf, sizeof buf, "conn row %d has non-integral endpoint", detail); break;
    case kConnMissing: std::snprintf(buf, sizeof buf, "conn row %d references a missing node", detail); break;
    case kDupPair: return "duplicate connection pair";
    default: return "";
  }
  return buf;
}

cudaError_t launch_validate(const double* nodes, const double* conns, int P, const DevShape& sh, int32_t* codes,
                            int32_t* details, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  const size_t per_warp = align16(size_t(table_capacity(sh.N) + table_capacity(sh.C)) * 8);
  int warps = 4;
  while (warps > 1 && per_warp * warps > 96 * 1024) warps >>= 1;
  cudaError_t e = cudaFuncSetAttribute(k_validate, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(per_warp * warps));
  if (e != cudaSuccess) return e;
  k_validate<<<(P + warps - 1) / warps, 32 * warps, per_warp * warps, st>>>(nodes, conns, P, sh, codes, details,
                                                                           per_warp);
  return cudaGetLastError();
}

}  // namespace fnb

// ---- C ABI (include/flatneat_b200.h) -------------------------------------------
using namespace fnb;

#define VCK(expr)                                                  \
  do {                                                             \
    cudaError_t e_ = (expr);                                       \
    if (e_ != cudaSuccess) return fnb_cuda_error(ctx, e_, #expr);  \
  } while (0)

extern "C" {

int fnb_explain_invalid_d(fnb_ctx* ctx, const double* d_nodes, const double* d_conns, int P, int32_t* d_codes,
                          int32_t* d_details, void* stream) {
  if (P <= 0) return 0;
  VCK(cudaSetDevice(ctx->device));
  VCK(launch_validate(d_nodes, d_conns, P, ctx->sh, d_codes, d_details, static_cast<cudaStream_t>(stream)));
  ctx->launches++;
  return 0;
}

int fnb_explain_invalid(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P, int32_t* codes,
                        int32_t* details) {
  ctx->err.clear();
  ctx->err_index = -1;
  if (P <= 0) return 0;
  VCK(cudaSetDevice(ctx->device));
  const size_t nb = sizeof(double) * size_t(P) * ctx->L.N * kNodeCols;
  const size_t cb = sizeof(double) * size_t(P) * ctx->L.C * kConnCols;
  VCK(ctx->nodes.ensure(nb));
  VCK(ctx->conns.ensure(cb));
  VCK(ctx->misc.ensure(sizeof(int32_t) * 2 * size_t(P)));
  int32_t* dcodes = static_cast<int32_t*>(ctx->misc.p);
  VCK(cudaMemcpyAsync(ctx->nodes.p, pop_nodes, nb, cudaMemcpyHostToDevice, ctx->stream));
  VCK(cudaMemcpyAsync(ctx->conns.p, pop_conns, cb, cudaMemcpyHostToDevice, ctx->stream));
  if (int st = fnb_explain_invalid_d(ctx, static_cast<double*>(ctx->nodes.p), static_cast<double*>(ctx->conns.p), P,
                                     dcodes, dcodes + P, ctx->stream))
    return st;
  VCK(cudaMemcpyAsync(codes, dcodes, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, ctx->stream));
  if (details) VCK(cudaMemcpyAsync(details, dcodes + P, sizeof(int32_t) * P, cudaMemcpyDeviceToHost, ctx->stream));
  VCK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int fnb_explain_message(int code, int detail, char* buf, size_t n) {
  const std::string m = validate_message(code, detail);
  if (buf && n) {
    std::snprintf(buf, n, "%s", m.c_str());
  }
  return int(m.size());
}

}  // extern "C"
