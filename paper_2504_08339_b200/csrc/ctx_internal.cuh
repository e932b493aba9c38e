// ctx_internal.cuh -- the fnb_ctx object behind the C ABI (shared by the
// translation units that implement it).
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <algorithm>

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

// Persistent host threads for memcpy from pageable memory into pinned
// staging buffers (fnb_evaluate / fnb_batch_forward with ordinary host
// arrays): one copy is split into >= 1 MB parts that the workers and the
// calling thread take in turn.
class CopyPool {
 public:
  explicit CopyPool(int threads) {
    for (int i = 0; i < threads; ++i) th_.emplace_back([this] { run(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(void* dst, const void* src, size_t n) {
    const size_t part = size_t(1) << 20;
    const size_t parts = (n + part - 1) / part;
    if (parts <= 1 || th_.empty()) {
      std::memcpy(dst, src, n);
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      n_ = n;
      part_ = part;
      parts_ = parts;
      next_.store(0);
      left_ = parts;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [this] { return left_ == 0; });
  }

 private:
  void work() {
    for (;;) {
      const size_t i = next_.fetch_add(1);
      if (i >= parts_) return;
      const size_t off = i * part_;
      std::memcpy(dst_ + off, src_ + off, std::min(part_, n_ - off));
      std::lock_guard<std::mutex> g(m_);
      if (--left_ == 0) done_.notify_all();
    }
  }
  void run() {
    size_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_ = 0, part_ = 0, parts_ = 0, left_ = 0, gen_ = 0;
  std::atomic<size_t> next_{0};
  bool stop_ = false;
};

// Pinned bounce buffers for pageable host inputs (a ring of kSlots chunks).
struct HostStage {
  static constexpr int kSlots = 3;
  void* buf[kSlots] = {};
  size_t cap = 0;
  cudaEvent_t free_ev[kSlots] = {};  // the slot's DMA finished
  CopyPool* pool = nullptr;
  cudaError_t ensure(size_t bytes) {
    if (!pool) pool = new CopyPool(int(std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2))));
    if (!free_ev[0])
      for (auto& e : free_ev) {
        cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        if (r != cudaSuccess) return r;
      }
    if (bytes <= cap) return cudaSuccess;
    for (auto& b : buf)
      if (b) {
        cudaFreeHost(b);
        b = nullptr;
      }
    cap = 0;
    for (auto& b : buf) {
      cudaError_t r = cudaMallocHost(&b, bytes);
      if (r != cudaSuccess) return r;
    }
    cap = bytes;
    return cudaSuccess;
  }
  void release() {
    for (auto& b : buf)
      if (b) cudaFreeHost(b);
    for (auto& e : free_ev)
      if (e) cudaEventDestroy(e);
    delete pool;
    *this = HostStage{};
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
  HostStage stage;
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
