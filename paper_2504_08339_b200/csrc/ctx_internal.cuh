// ctx_internal.cuh -- the fnb_ctx object behind the C ABI (shared by the
// translation units that implement it).
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
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

// Persistent host threads for the host side of fnb_evaluate /
// fnb_batch_forward: packing the FP64 genome rows into the transfer rows of
// K1 (pack_genomes below) and memcpy from pageable memory into pinned staging
// buffers.  A job is split into parts that the workers and the calling
// thread take in turn; run() returns when every part is done.
class CopyPool {
 public:
  explicit CopyPool(int threads) {
    for (int i = 0; i < threads; ++i) th_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // f(i) for i in [0, parts); the calling thread takes parts too
  void run(size_t parts, std::function<void(size_t)> f) {
    if (parts == 0) return;
    if (parts == 1 || th_.empty()) {
      for (size_t i = 0; i < parts; ++i) f(i);
      return;
    }
    start(parts, std::move(f));
    work();
    wait();
  }
  // the same on the workers only, returning at once (wait() joins): the
  // caller enqueues GPU work meanwhile
  void start(size_t parts, std::function<void(size_t)> f) {
    if (th_.empty()) {
      for (size_t i = 0; i < parts; ++i) f(i);
      return;
    }
    {
      std::lock_guard<std::mutex> g(m_);
      job_ = std::move(f);
      parts_ = parts;
      next_.store(0);
      left_ = parts;
      ++gen_;
    }
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [this] { return left_ == 0; });
  }
  void copy(void* dst, const void* src, size_t n) {
    const size_t part = size_t(1) << 20;
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    run((n + part - 1) / part, [=](size_t i) {
      const size_t off = i * part;
      std::memcpy(d + off, s + off, std::min(part, n - off));
    });
  }
  int threads() const { return int(th_.size()) + 1; }

 private:
  void work() {
    for (;;) {
      const size_t i = next_.fetch_add(1);
      if (i >= parts_) return;
      job_(i);
      std::lock_guard<std::mutex> g(m_);
      if (--left_ == 0) done_.notify_all();
    }
  }
  void loop() {
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
  std::function<void(size_t)> job_;
  size_t parts_ = 0, left_ = 0, gen_ = 0;
  std::atomic<size_t> next_{0};
  bool stop_ = false;
};

// int(x) as K1's conversions compute it on the device (F2I.S32.F64.TRUNC):
// NaN -> INT32_MIN (measured: "aggregation id -2147483648"), out-of-range
// values saturate
inline int32_t dev_int(double x) {
  if (x != x) return -2147483647 - 1;
  if (x >= 2147483647.0) return 2147483647;
  if (x <= -2147483648.0) return -2147483647 - 1;
  return int32_t(x);
}

// Genomes [g0, g1) of the FP64 population rows -> packed transfer rows
// (fnb::PackedLayout blocks from `out`).  Returns false if a non-empty node's
// activation or aggregation id does not fit a byte (the caller then sends the
// FP64 rows: only an invalid genome can have one).
inline bool pack_genomes(const double* nodes, const double* conns, int N, int C, size_t g0, size_t g1,
                         uint8_t* out) {
  const fnb::PackedLayout pk(N, C);
  bool ok = true;
  for (size_t g = g0; g < g1; ++g) {
    const double* n = nodes + g * size_t(N) * fnb::kNodeCols;
    const double* c = conns + g * size_t(C) * fnb::kConnCols;
    uint8_t* b = out + (g - g0) * pk.bytes;
    int32_t* key = reinterpret_cast<int32_t*>(b + pk.key);
    float* bias = reinterpret_cast<float*>(b + pk.bias);
    float* resp = reinterpret_cast<float*>(b + pk.resp);
    for (int r = 0; r < N; ++r) {
      const double* x = n + size_t(r) * fnb::kNodeCols;
      const bool ne = !(x[0] != x[0]);
      const int32_t ac = dev_int(x[fnb::kAct]), ag = dev_int(x[fnb::kAgg]);
      ok &= !ne || (uint32_t(ac) < 256u && uint32_t(ag) < 256u);
      key[r] = dev_int(x[fnb::kKey]);
      bias[r] = float(x[fnb::kBias]);
      resp[r] = float(x[fnb::kResp]);
      b[pk.act + r] = uint8_t(ac);
      b[pk.agg + r] = uint8_t(ag);
      b[pk.nflag + r] = uint8_t(ne);
    }
    int32_t* cin = reinterpret_cast<int32_t*>(b + pk.cin);
    int32_t* cout = reinterpret_cast<int32_t*>(b + pk.cout);
    float* w = reinterpret_cast<float*>(b + pk.w);
    for (int r = 0; r < C; ++r) {
      const double* x = c + size_t(r) * fnb::kConnCols;
      cin[r] = dev_int(x[fnb::kIn]);
      cout[r] = dev_int(x[fnb::kOut]);
      w[r] = float(x[fnb::kW]);
      b[pk.cflag + r] = uint8_t(!(x[fnb::kIn] != x[fnb::kIn])) | uint8_t((x[fnb::kEn] == 1.0) << 1);
    }
  }
  return ok;
}

// Pinned bounce buffers for pageable host inputs (a ring of kSlots chunks).
struct HostStage {
  static constexpr int kSlots = 3;
  void* buf[kSlots] = {};
  size_t cap = 0;
  cudaEvent_t free_ev[kSlots] = {};  // the slot's DMA finished
  CopyPool* pool = nullptr;
  cudaError_t ensure(size_t bytes) {
    if (!pool) pool = new CopyPool(int(std::max(1u, std::thread::hardware_concurrency()) - 1));
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
  DevBuf nodes, conns, nets, X, Y, fit, out, partial, misc, scratch, flags, hyper, packed;
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
