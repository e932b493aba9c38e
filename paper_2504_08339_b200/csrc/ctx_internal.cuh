// ctx_internal.cuh -- the fnb_ctx object behind the C ABI (shared by the
// translation units that implement it).
#pragma once
#include <string>

#include "fnb_common.cuh"

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct fnb_ctx {
  int device = 0;
  fnb::DevShape sh{};
  fnb::NetLayout L{0, 0, 0, 0};
  std::string err;
  int err_index = -1;
  long long launches = 0;
  cudaStream_t stream = nullptr;
  // host-layer pipeline: population chunks go up on copy_stream while the
  // previous chunk is transformed and evaluated on `stream`
  cudaStream_t copy_stream = nullptr;
  static constexpr int kMaxChunks = 32;
  cudaEvent_t chunk_ev[kMaxChunks + 1] = {};
  DevBuf nodes, conns, nets, X, Y, fit, out, partial, misc, scratch, flags, hyper;
};

// errors.hpp:33-57
inline const char* fnb_errc_name(int c) {
  static const char* names[] = {
      "unknown_function", "genome_full", "duplicate_key", "duplicate_conn",
      "dangling_endpoint", "key_not_found", "protected_node", "attr_out_of_range",
      "shape_mismatch", "corrupt_row", "cycle_detected", "non_finite_input",
      "non_finite_state", "empty_aggregation", "empty_dataset", "parse_error",
      "version_unsupported", "limits_too_small", "config_error", "eval_error"};
  return (c >= 0 && c < 20) ? names[c] : "unknown";
}

inline int fnb_set_error(fnb_ctx* ctx, int code, const std::string& detail, int index) {
  ctx->err = std::string(fnb_errc_name(code)) + ": " + detail;
  ctx->err_index = index;
  return 1 + code;
}

inline int fnb_cuda_error(fnb_ctx* ctx, cudaError_t e, const char* what) {
  if (ctx) {
    ctx->err = std::string("eval_error: CUDA ") + cudaGetErrorString(e) + " at " + what;
    ctx->err_index = -1;
  }
  return 1 + FNB_E_EVAL_ERROR;
}
