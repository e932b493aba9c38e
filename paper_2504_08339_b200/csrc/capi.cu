#include <cmath>
// capi.cu -- extern "C" boundary (include/flatneat_b200.h): contexts, the
// synchronous host layer mirroring the reference free functions, and the
// asynchronous device layer.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <chrono>
#include <vector>

#include "fnb_common.cuh"
#include "ctx_internal.cuh"

namespace fnb {
// host launchers (transform.cu / forward.cu)
cudaError_t launch_transform(const double* n, const double* c, int P, uint8_t* nets, const NetLayout& L,
                             const DevShape& sh, cudaStream_t st);
cudaError_t launch_transform_packed(const uint8_t* packed, int P, uint8_t* nets, const NetLayout& L,
                                    const DevShape& sh, cudaStream_t st);
cudaError_t launch_describe_cycle(const double* n, const double* c, const uint8_t* net, const NetLayout& L,
                                  int* path, cudaStream_t st);
cudaError_t launch_first_error(const uint8_t* nets, size_t stride, int P, int* out, cudaStream_t st);
cudaError_t launch_net_order(const uint8_t* nets, const NetLayout& L, int P, int32_t* order, int32_t* count,
                             cudaStream_t st);
int launch_forward(const void* nets, NetLayout L, int P, const float* X, const float* Y, int B,
                   int fit_kind, double offset, double* fitness, double* out, double* partial_buf,
                   size_t partial_cap, int uniform_agg, int uniform_act, cudaStream_t st, long long* launches);
size_t forward_partial_needed(NetLayout L, int P, int B);
void set_forward_spt(int spt);
void set_forward_tuning(int spt, int max_cols, int rows_pct, int group_kb);
void set_forward_recs_pct(int pct);
cudaError_t launch_to_float(const double* src, float* dst, size_t n, int* bad, cudaStream_t st);
}  // namespace fnb

using namespace fnb;

namespace {

const char* errc_name(int c) {  // errors.hpp:33-57
  static const char* names[] = {
      "unknown_function", "genome_full", "duplicate_key", "duplicate_conn",
      "dangling_endpoint", "key_not_found", "protected_node", "attr_out_of_range",
      "shape_mismatch", "corrupt_row", "cycle_detected", "non_finite_input",
      "non_finite_state", "empty_aggregation", "empty_dataset", "parse_error",
      "version_unsupported", "limits_too_small", "config_error", "eval_error"};
  return (c >= 0 && c < 20) ? names[c] : "unknown";
}

}  // namespace

static int fnb_cuda_fail_ctx(fnb_ctx* ctx, cudaError_t e, const char* what) {
  if (ctx) {
    ctx->err = std::string("eval_error: CUDA ") + cudaGetErrorString(e) + " at " + what;
    ctx->err_index = -1;
  }
  return 1 + FNB_E_EVAL_ERROR;
}

#define CK(expr)                                                 \
  do {                                                           \
    cudaError_t e_ = (expr);                                     \
    if (e_ != cudaSuccess) return fnb_cuda_fail_ctx(ctx, e_, #expr); \
  } while (0)

static int set_err(fnb_ctx* ctx, int code, const std::string& detail, int index) {
  ctx->err = std::string(errc_name(code)) + ": " + detail;
  ctx->err_index = index;
  return 1 + code;
}

extern "C" {

int fnb_abi_version(void) { return FNB_ABI_VERSION; }

int fnb_ctx_create(const fnb_shape* shape, const fnb_schema* schema, int device, fnb_ctx** out) {
  if (!shape || !schema || !out) return 1 + FNB_E_CONFIG_ERROR;
  *out = nullptr;
  if (shape->max_nodes < 1 || shape->max_nodes > FNB_MAX_NODES_LIMIT || shape->max_conns < 1 ||
      shape->max_conns > 65535 || shape->num_inputs < 0 || shape->num_inputs > 32 ||
      shape->num_outputs < 0 || shape->num_outputs > 32)
    return 1 + FNB_E_LIMITS_TOO_SMALL;
  if (schema->n_act < 1 || schema->n_act > 8 || schema->n_agg < 1 || schema->n_agg > 8)
    return 1 + FNB_E_CONFIG_ERROR;
  for (int i = 0; i < schema->n_act; ++i)
    if (schema->act[i] < FNB_ACT_IDENTITY || schema->act[i] > FNB_ACT_SIN) return 1 + FNB_E_UNKNOWN_FUNCTION;
  for (int i = 0; i < schema->n_agg; ++i)
    if (schema->agg[i] < FNB_AGG_SUM || schema->agg[i] > FNB_AGG_MEAN) return 1 + FNB_E_UNKNOWN_FUNCTION;
  auto* ctx = new fnb_ctx();
  ctx->device = device;
  DevShape& sh = ctx->sh;
  sh.N = shape->max_nodes;
  sh.C = shape->max_conns;
  sh.I = shape->num_inputs;
  sh.O = shape->num_outputs;
  sh.n_act = schema->n_act;
  sh.n_agg = schema->n_agg;
  for (int i = 0; i < 8; ++i) {
    sh.act[i] = uint8_t(i < schema->n_act ? schema->act[i] : 0);
    sh.agg[i] = uint8_t(i < schema->n_agg ? schema->agg[i] : 0);
  }
  sh.default_act = schema->default_act;
  sh.default_agg = schema->default_agg;
  for (int i = 0; i < sh.I; ++i) sh.input_keys[i] = shape->input_keys[i];
  for (int i = 0; i < sh.O; ++i) sh.output_keys[i] = shape->output_keys[i];
  ctx->L = NetLayout(sh.N, sh.C, sh.I, sh.O);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return 1 + FNB_E_EVAL_ERROR;
  }
  *out = ctx;
  return 0;
}

void fnb_ctx_destroy(fnb_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (DevBuf* b : {&ctx->nodes, &ctx->conns, &ctx->nets, &ctx->X, &ctx->Y, &ctx->fit, &ctx->out,
                    &ctx->partial, &ctx->misc, &ctx->scratch})
    b->release();
  ctx->flags.release();
  ctx->hyper.release();
  ctx->packed.release();
  ctx->stage.release();
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->copy_stream) {
    cudaStreamDestroy(ctx->copy_stream);
    for (auto& e : ctx->chunk_ev) cudaEventDestroy(e);
  }
  delete ctx;
}

const char* fnb_last_error(const fnb_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }
int fnb_last_error_index(const fnb_ctx* ctx) { return ctx ? ctx->err_index : -1; }
size_t fnb_net_bytes(const fnb_ctx* ctx) { return ctx ? ctx->L.bytes : 0; }
long long fnb_launch_count(const fnb_ctx* ctx) { return ctx ? ctx->launches : 0; }
void fnb_set_forward_spt(int spt) { set_forward_spt(spt); }
void fnb_set_forward_tuning(int spt, int max_cols, int rows_pct, int group_kb) {
  set_forward_tuning(spt, max_cols, rows_pct, group_kb);
}

void fnb_set_forward_recs_pct(int pct) { set_forward_recs_pct(pct); }

// host transfer format (fnb_set_host_transfer_packed; FNB_H2D_PACK=0 starts it off)
static std::atomic<bool> g_host_pack{[] {
  const char* e = std::getenv("FNB_H2D_PACK");
  return !(e && std::atoi(e) == 0);
}()};

void fnb_set_host_transfer_packed(int on) { g_host_pack.store(on != 0); }

// ---- device layer ------------------------------------------------------

int fnb_transform_d(fnb_ctx* ctx, const double* d_nodes, const double* d_conns, int P, void* d_nets,
                    void* stream) {
  if (P <= 0) return 0;
  CK(cudaSetDevice(ctx->device));
  CK(launch_transform(d_nodes, d_conns, P, static_cast<uint8_t*>(d_nets), ctx->L, ctx->sh,
                      static_cast<cudaStream_t>(stream)));
  ctx->launches++;
  return 0;
}

int fnb_net_order_d(fnb_ctx* ctx, const void* d_nets, int P, int32_t* d_order, int32_t* d_count,
                    void* stream) {
  if (P <= 0) return 0;
  CK(cudaSetDevice(ctx->device));
  CK(launch_net_order(static_cast<const uint8_t*>(d_nets), ctx->L, P, d_order, d_count,
                      static_cast<cudaStream_t>(stream)));
  ctx->launches++;
  return 0;
}

int fnb_check_nets_d(fnb_ctx* ctx, const double* d_nodes, const double* d_conns, const void* d_nets,
                     int P, void* stream) {
  ctx->err.clear();
  ctx->err_index = -1;
  if (P <= 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  const int N = ctx->L.N;
  CK(ctx->misc.ensure(sizeof(int) * size_t(N + 8)));
  int* d_first = static_cast<int*>(ctx->misc.p);
  const int big = 0x7fffffff;
  CK(cudaMemcpyAsync(d_first, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  CK(launch_first_error(static_cast<const uint8_t*>(d_nets), ctx->L.bytes, P, d_first, st));
  ctx->launches++;
  int first = big;
  CK(cudaMemcpyAsync(&first, d_first, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (first == big) return 0;
  NetHeader h;
  const uint8_t* net = static_cast<const uint8_t*>(d_nets) + size_t(first) * ctx->L.bytes;
  CK(cudaMemcpy(&h, net, sizeof(h), cudaMemcpyDeviceToHost));
  const int code = h.status - 1;
  char buf[64];
  switch (h.err_kind) {
    case kErrActId: std::snprintf(buf, sizeof buf, "activation id %d out of range", h.err_a); break;
    case kErrAggId: std::snprintf(buf, sizeof buf, "aggregation id %d out of range", h.err_a); break;
    case kErrInputKey: std::snprintf(buf, sizeof buf, "input key %d", h.err_a); break;
    case kErrOutputKey: std::snprintf(buf, sizeof buf, "output key %d", h.err_a); break;
    case kErrConn: std::snprintf(buf, sizeof buf, "conn (%d, %d)", h.err_a, h.err_b); break;
    case kErrCycle: {
      int* d_path = d_first + 1;
      CK(launch_describe_cycle(d_nodes + size_t(first) * N * kNodeCols,
                               d_conns + size_t(first) * ctx->L.C * kConnCols, net, ctx->L, d_path, st));
      ctx->launches++;
      std::vector<int> path(size_t(N) + 2);
      CK(cudaMemcpyAsync(path.data(), d_path, sizeof(int) * (size_t(N) + 2), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::string s = "cycle ";
      if (path[0] < 0) {
        s += "unlocatable cycle";
      } else {
        for (int i = 0; i < path[0]; ++i) {
          if (i) s += "->";
          s += std::to_string(path[1 + i]);
        }
      }
      return set_err(ctx, code, s, first);
    }
    default: std::snprintf(buf, sizeof buf, "status %d", h.status);
  }
  return set_err(ctx, code, buf, first);
}

int fnb_forward_d(fnb_ctx* ctx, const void* d_nets, int P, const float* d_X, const float* d_Y, int batch,
                  int fitness_kind, double fitness_offset, double* d_fitness, double* d_out, void* stream) {
  if (P <= 0 || batch <= 0) return 0;
  if (fitness_kind != FNB_FIT_NONE && (!d_Y || !d_fitness)) return set_err(ctx, FNB_E_CONFIG_ERROR, "fitness needs targets and output", -1);
  CK(cudaSetDevice(ctx->device));
  CK(ctx->partial.ensure(forward_partial_needed(ctx->L, P, batch)));
  return launch_forward(d_nets, ctx->L, P, d_X, d_Y, batch, fitness_kind, fitness_offset, d_fitness, d_out,
                        static_cast<double*>(ctx->partial.p), ctx->partial.cap,
                        ctx->sh.n_agg == 1 ? int(ctx->sh.agg[0]) : -1, ctx->sh.n_act == 1 ? int(ctx->sh.act[0]) : -1,
                        static_cast<cudaStream_t>(stream), &ctx->launches)
             ? fnb_cuda_fail_ctx(ctx, cudaGetLastError(), "forward launch")
             : 0;
}

// ---- host layer ----------------------------------------------------------

static int upload_pop(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P) {
  const size_t nb = sizeof(double) * size_t(P) * ctx->L.N * kNodeCols;
  const size_t cb = sizeof(double) * size_t(P) * ctx->L.C * kConnCols;
  CK(ctx->nodes.ensure(nb));
  CK(ctx->conns.ensure(cb));
  CK(ctx->nets.ensure(ctx->L.bytes * size_t(P)));
  CK(cudaMemcpyAsync(ctx->nodes.p, pop_nodes, nb, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->conns.p, pop_conns, cb, cudaMemcpyHostToDevice, ctx->stream));
  return 0;
}

static int transform_and_check(fnb_ctx* ctx, int P) {
  int st = fnb_transform_d(ctx, static_cast<double*>(ctx->nodes.p), static_cast<double*>(ctx->conns.p), P,
                           ctx->nets.p, ctx->stream);
  if (st) return st;
  return fnb_check_nets_d(ctx, static_cast<double*>(ctx->nodes.p), static_cast<double*>(ctx->conns.p),
                          ctx->nets.p, P, ctx->stream);
}

int fnb_transform(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P, int32_t* order_out,
                  int32_t* order_count_out) {
  ctx->err.clear();
  ctx->err_index = -1;
  if (P <= 0) return 0;
  CK(cudaSetDevice(ctx->device));
  int st = upload_pop(ctx, pop_nodes, pop_conns, P);
  if (!st) st = transform_and_check(ctx, P);
  if (st) return st;
  if (order_out || order_count_out) {
    const size_t ob = sizeof(int32_t) * size_t(P) * ctx->L.N, cb = sizeof(int32_t) * size_t(P);
    CK(ctx->out.ensure(ob + cb));
    int32_t* d_order = static_cast<int32_t*>(ctx->out.p);
    int32_t* d_cnt = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ctx->out.p) + ob);
    st = fnb_net_order_d(ctx, ctx->nets.p, P, d_order, d_cnt, ctx->stream);
    if (st) return st;
    if (order_out) CK(cudaMemcpyAsync(order_out, d_order, ob, cudaMemcpyDeviceToHost, ctx->stream));
    if (order_count_out) CK(cudaMemcpyAsync(order_count_out, d_cnt, cb, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return 0;
}

// Lazily created copy stream + chunk events of the host-layer pipeline.
static int ensure_pipeline(fnb_ctx* ctx) {
  if (ctx->copy_stream) return 0;
  CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  for (auto& e : ctx->chunk_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return 0;
}

// Host-buffer evaluation (batch_forward network.hpp:294-330 + the fitness of
// SPEC.md:441-458).  The population crosses PCIe in chunks on copy_stream;
// chunk k is transformed (K1) and evaluated (K2) on the compute stream as
// soon as its copy lands, so the transfer of chunk k+1 overlaps the kernels
// of chunk k.  Per-genome fitness is partition invariant (forward.cu), so
// the chunking does not change a bit of the result.  Errors are collected on
// the device and read once at the end, in the reference's order: the lowest
// failing genome's transform error (network.hpp:122-220), then a non-finite
// input (network.hpp:245-246).
//
// Transfer format.  Pageable host arrays (a std::vector caller) are staged
// through pinned buffers anyway; by default the host threads pack each chunk
// into K1's transfer rows there (PackedLayout: 0.40 of the bytes at C2,
// converted exactly as K1 converts the FP64 rows) and only those cross PCIe;
// K1 reads them (launch_transform_packed): C2 e2e 2.3 -> 4.4 G evals/s.
// Pinned arrays go up by DMA as they are.  The FP64 rows go up for a packed
// call only to rebuild an error message, or for the whole call when a node's
// act / agg id does not fit the packed byte.  fnb_set_host_transfer_packed(0)
// (or FNB_H2D_PACK=0) stages the FP64 rows.
static int evaluate_impl(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P,
                         const double* inputs, const double* targets, int batch, int kind, double offset,
                         double* fitness_out, double* out, bool allow_pack = true) {
  ctx->err.clear();
  ctx->err_index = -1;
  if (P <= 0) return 0;
  CK(cudaSetDevice(ctx->device));
  if (int st = ensure_pipeline(ctx)) return st;
  const int N = ctx->L.N, Cm = ctx->L.C, O = ctx->L.O;
  const size_t nrow = sizeof(double) * size_t(N) * kNodeCols, crow = sizeof(double) * size_t(Cm) * kConnCols;
  auto pageable = [](const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
      cudaGetLastError();
      return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
  };
  // Pageable arrays are packed (they are staged through host memory anyway:
  // ~2x the e2e at C2).  Pinned arrays go up by DMA as they are: packing all
  // or a share of their chunks on the host threads measured 2.2-3.3 ms per C2
  // call against 2.23 ms (scripts/h2d_trace.sh, round 2) -- the host's memory
  // bandwidth bounds the DMA and the packers together.
  const bool src_pageable = pageable(pop_nodes) || pageable(pop_conns);
  const bool pack = allow_pack && g_host_pack.load() && src_pageable;
  auto is_pk = [&](int) { return pack; };
  const PackedLayout pkl(N, Cm);
  if (!pack) {
    CK(ctx->nodes.ensure(nrow * size_t(P)));
    CK(ctx->conns.ensure(crow * size_t(P)));
  } else {
    CK(ctx->packed.ensure(pkl.bytes * size_t(P)));
  }
  CK(ctx->nets.ensure(ctx->L.bytes * size_t(P)));
  CK(ctx->flags.ensure(4 * sizeof(int)));
  int* d_flags = static_cast<int*>(ctx->flags.p);  // [0] first failing genome, [1] non-finite X, [2] Y
  static const int kInit[4] = {0x7fffffff, 0, 0, 0};
  CK(cudaMemcpyAsync(d_flags, kInit, sizeof(kInit), cudaMemcpyHostToDevice, ctx->stream));
  // X and Y go up as doubles and are narrowed on the device
  auto up = [&](DevBuf& dst, const double* src, size_t n, int* bad) -> int {
    CK(dst.ensure(n * sizeof(float) + n * sizeof(double) + 16));
    double* d_tmp = reinterpret_cast<double*>(static_cast<uint8_t*>(dst.p) + ((n * sizeof(float) + 15) & ~size_t(15)));
    CK(cudaMemcpyAsync(d_tmp, src, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(launch_to_float(d_tmp, static_cast<float*>(dst.p), n, bad, ctx->stream));
    ctx->launches++;
    return 0;
  };
  if (int st = up(ctx->X, inputs, size_t(batch) * ctx->L.I, d_flags + 1)) return st;
  if (kind != FNB_FIT_NONE)
    if (int st = up(ctx->Y, targets, size_t(batch) * O, d_flags + 2)) return st;
  double* d_out = nullptr;
  double* d_fit = nullptr;
  if (out) {
    CK(ctx->out.ensure(sizeof(double) * size_t(P) * batch * O));
    d_out = static_cast<double*>(ctx->out.p);
  }
  if (kind != FNB_FIT_NONE) {
    CK(ctx->fit.ensure(sizeof(double) * size_t(P)));
    d_fit = static_cast<double*>(ctx->fit.p);
  }
  // chunks of ~chunk_mb MB, at most kMaxChunks.  8 MB measured best at C2
  // (scripts/sweep_h2d.py): smaller chunks leave K1/K2 too little work per
  // launch, larger ones lengthen the pipeline fill; a second copy stream
  // only contends for the link.  FNB_H2D_CHUNK_MB overrides (tuning).
  static const int chunk_mb = [] {
    const char* e = std::getenv("FNB_H2D_CHUNK_MB");
    const int v = e ? std::atoi(e) : 8;
    return v >= 1 && v <= 256 ? v : 8;
  }();
  const size_t total = (nrow + crow) * size_t(P);
  const int chunks = int(std::max<size_t>(
      1, std::min<size_t>(std::min<size_t>(fnb_ctx::kMaxChunks, size_t(P)), total / (size_t(chunk_mb) << 20))));
  auto lo_of = [&](int k) { return int((long long)P * k / chunks); };
  // pageable host arrays (what a std::vector caller passes) go through pinned
  // bounce buffers: the host threads copy chunk k+1 while chunk k is on the
  // wire and chunk k-1 in K1/K2 (a plain cudaMemcpyAsync from pageable memory
  // is staged synchronously by the driver)
  const bool staged = pack || src_pageable;
  if (staged) {
    size_t most = 0;
    for (int k = 0; k < chunks; ++k)
      most = std::max(most, size_t(lo_of(k + 1) - lo_of(k)) * (is_pk(k) ? pkl.bytes : nrow + crow));
    CK(ctx->stage.ensure(most));
  }
  bool pack_ok = true;
  static const bool trace = std::getenv("FNB_H2D_TRACE") != nullptr;  // per-call host timing (stderr)
  double t_copy = 0.0, t_launch = 0.0;
  const auto call_t0 = std::chrono::steady_clock::now();
  std::atomic<bool> pack_good{true};
  bool next_ready = false;  // the chunk about to be enqueued was packed by the previous iteration
  // the pool workers pack chunk k into its staging slot (asynchronously; pool->wait() joins)
  auto pack_chunk = [&](int k) {
    const size_t lo = size_t(lo_of(k)), hi = size_t(lo_of(k + 1));
    uint8_t* b = static_cast<uint8_t*>(ctx->stage.buf[k % HostStage::kSlots]);
    constexpr size_t kPart = 16;  // genomes per pool part
    ctx->stage.pool->start((hi - lo + kPart - 1) / kPart, [=, &pack_good](size_t i) {
      const size_t g0 = lo + i * kPart, g1 = std::min(hi, g0 + kPart);
      if (!pack_genomes(pop_nodes, pop_conns, N, Cm, g0, g1, b + (g0 - lo) * pkl.bytes)) pack_good.store(false);
    });
  };
  struct PoolJoin {  // no early return leaves a packing job running on this frame's data
    CopyPool* p;
    ~PoolJoin() {
      if (p) p->wait();
    }
  } pool_join{pack ? ctx->stage.pool : nullptr};
  // GPU-side timeline of the call (FNB_H2D_TRACE): first copy issued, last copy landed, last kernel done
  cudaEvent_t tev[3] = {};
  if (trace)
    for (auto& e : tev) CK(cudaEventCreate(&e));
  // the copies must not overwrite buffers still read by earlier work on the compute stream
  CK(cudaEventRecord(ctx->chunk_ev[fnb_ctx::kMaxChunks], ctx->stream));
  CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->chunk_ev[fnb_ctx::kMaxChunks], 0));
  if (trace) CK(cudaEventRecord(tev[0], ctx->copy_stream));
  uint8_t* dn = static_cast<uint8_t*>(ctx->nodes.p);
  uint8_t* dc = static_cast<uint8_t*>(ctx->conns.p);
  uint8_t* nets = static_cast<uint8_t*>(ctx->nets.p);
  for (int k = 0; k < chunks; ++k) {
    const int lo = lo_of(k), n = lo_of(k + 1) - lo;
    cudaStream_t cs = ctx->copy_stream;
    const uint8_t* hn = reinterpret_cast<const uint8_t*>(pop_nodes) + size_t(lo) * nrow;
    const uint8_t* hc = reinterpret_cast<const uint8_t*>(pop_conns) + size_t(lo) * crow;
    uint8_t* dp = static_cast<uint8_t*>(ctx->packed.p) + size_t(lo) * pkl.bytes;
    const bool pk = is_pk(k);
    if (pk) {
      // chunk k is packed into its slot (by the previous iteration, or here);
      // the workers pack the next packed chunk while this thread enqueues k
      if (!next_ready) {
        CK(cudaEventSynchronize(ctx->stage.free_ev[k % HostStage::kSlots]));
        pack_chunk(k);
        ctx->stage.pool->wait();
      }
      if (!pack_good.load()) {
        pack_ok = false;
        break;
      }
    }
    next_ready = false;
    const bool prefetch = k + 1 < chunks && is_pk(k + 1);
    if (prefetch) {
      CK(cudaEventSynchronize(ctx->stage.free_ev[(k + 1) % HostStage::kSlots]));  // that slot's last DMA has left
      pack_chunk(k + 1);
    }
    if (pk) {
      CK(cudaMemcpyAsync(dp, ctx->stage.buf[k % HostStage::kSlots], size_t(n) * pkl.bytes, cudaMemcpyHostToDevice,
                         cs));
    } else {
      if (src_pageable) {
        const int slot = k % HostStage::kSlots;
        CK(cudaEventSynchronize(ctx->stage.free_ev[slot]));  // that slot's previous chunk has left
        uint8_t* b = static_cast<uint8_t*>(ctx->stage.buf[slot]);
        ctx->stage.pool->copy(b, hn, size_t(n) * nrow);
        ctx->stage.pool->copy(b + size_t(n) * nrow, hc, size_t(n) * crow);
        hn = b;
        hc = b + size_t(n) * nrow;
      }
      const auto tm0 = std::chrono::steady_clock::now();
      // pinned arrays: every node row in the first copy (one DMA instead of one
      // per chunk: ~4.5 us each on this link), the connection rows per chunk
      if (src_pageable)
        CK(cudaMemcpyAsync(dn + size_t(lo) * nrow, hn, size_t(n) * nrow, cudaMemcpyHostToDevice, cs));
      else if (k == 0)
        CK(cudaMemcpyAsync(dn, pop_nodes, size_t(P) * nrow, cudaMemcpyHostToDevice, cs));
      CK(cudaMemcpyAsync(dc + size_t(lo) * crow, hc, size_t(n) * crow, cudaMemcpyHostToDevice, cs));
      if (trace) t_copy += std::chrono::duration<double>(std::chrono::steady_clock::now() - tm0).count();
    }
    if (pk || src_pageable) CK(cudaEventRecord(ctx->stage.free_ev[k % HostStage::kSlots], cs));
    CK(cudaEventRecord(ctx->chunk_ev[k], cs));
    if (trace && k == chunks - 1) CK(cudaEventRecord(tev[1], cs));
    // chunk k's K1 + K2 on the compute stream as soon as its copy lands
    CK(cudaStreamWaitEvent(ctx->stream, ctx->chunk_ev[k], 0));
    int st = 0;
    const auto tk0 = std::chrono::steady_clock::now();
    if (pk) {
      CK(launch_transform_packed(dp, n, nets + size_t(lo) * ctx->L.bytes, ctx->L, ctx->sh, ctx->stream));
      ctx->launches++;
    } else {
      st = fnb_transform_d(ctx, reinterpret_cast<const double*>(dn + size_t(lo) * nrow),
                           reinterpret_cast<const double*>(dc + size_t(lo) * crow), n,
                           nets + size_t(lo) * ctx->L.bytes, ctx->stream);
    }
    if (st) return st;
    // genomes that failed K1 carry no records: K2 skips them
    st = fnb_forward_d(ctx, nets + size_t(lo) * ctx->L.bytes, n, static_cast<float*>(ctx->X.p),
                       kind != FNB_FIT_NONE ? static_cast<float*>(ctx->Y.p) : nullptr, batch, kind, offset,
                       d_fit ? d_fit + lo : nullptr, d_out ? d_out + size_t(lo) * batch * O : nullptr, ctx->stream);
    if (trace) t_launch += std::chrono::duration<double>(std::chrono::steady_clock::now() - tk0).count();
    if (prefetch) {
      ctx->stage.pool->wait();  // chunk k+1 is packed
      next_ready = true;
    }
    if (st) return st;
  }
  if (!pack_ok) {  // an act / agg id beyond a byte: the whole call on the FP64 rows
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaStreamSynchronize(ctx->copy_stream));
    return evaluate_impl(ctx, pop_nodes, pop_conns, P, inputs, targets, batch, kind, offset, fitness_out, out,
                         false);
  }
  if (trace) CK(cudaEventRecord(tev[2], ctx->stream));
  CK(launch_first_error(nets, ctx->L.bytes, P, d_flags, ctx->stream));
  ctx->launches++;
  int flags[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(flags, d_flags, sizeof(flags), cudaMemcpyDeviceToHost, ctx->stream));
  if (out)
    CK(cudaMemcpyAsync(out, d_out, sizeof(double) * size_t(P) * batch * O, cudaMemcpyDeviceToHost, ctx->stream));
  if (fitness_out)
    CK(cudaMemcpyAsync(fitness_out, d_fit, sizeof(double) * size_t(P), cudaMemcpyDeviceToHost, ctx->stream));
  const auto sync_t0 = std::chrono::steady_clock::now();
  CK(cudaStreamSynchronize(ctx->stream));
  if (trace) {
    float dma = 0.f, all = 0.f;
    cudaEventElapsedTime(&dma, tev[0], tev[1]);
    cudaEventElapsedTime(&all, tev[0], tev[2]);
    std::fprintf(stderr, "  GPU: copies %.3f ms, copies + last K1/K2 %.3f ms\n", dma, all);
    for (auto& e : tev) cudaEventDestroy(e);
  }
  if (trace)
    std::fprintf(stderr, "evaluate P=%d chunks=%d packed %d: copies %.3f ms, K1/K2 launches %.3f ms, enqueue %.3f ms, wait %.3f ms\n", P, chunks,
                 int(pack), t_copy * 1e3, t_launch * 1e3, std::chrono::duration<double>(sync_t0 - call_t0).count() * 1e3,
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - sync_t0).count() * 1e3);
  if (flags[0] != 0x7fffffff) {  // rebuild the reference's message for the lowest failing genome
    if (pack) {  // from the FP64 rows, which only the error path uploads
      CK(ctx->nodes.ensure(nrow * size_t(P)));
      CK(ctx->conns.ensure(crow * size_t(P)));
      dn = static_cast<uint8_t*>(ctx->nodes.p);
      dc = static_cast<uint8_t*>(ctx->conns.p);
      CK(cudaMemcpy(dn, pop_nodes, nrow * size_t(P), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dc, pop_conns, crow * size_t(P), cudaMemcpyHostToDevice));
    }
    return fnb_check_nets_d(ctx, reinterpret_cast<const double*>(dn), reinterpret_cast<const double*>(dc), nets, P,
                            ctx->stream);
  }
  if (flags[1]) return set_err(ctx, FNB_E_NON_FINITE_INPUT, "input not finite", 0);  // network.hpp:245-246
  return 0;
}

int fnb_batch_forward(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P,
                      const double* inputs, int batch, double* out) {
  return evaluate_impl(ctx, pop_nodes, pop_conns, P, inputs, nullptr, batch, FNB_FIT_NONE, 0.0, nullptr, out);
}

int fnb_evaluate(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P, const double* inputs,
                 const double* targets, int batch, int fitness_kind, double fitness_offset, double* fitness_out) {
  if (fitness_kind == FNB_FIT_NONE) return set_err(ctx, FNB_E_CONFIG_ERROR, "fitness kind required", -1);
  // SPEC.md:458 (func_fit / xor): an empty dataset has no fitness
  if (batch <= 0) return set_err(ctx, FNB_E_EMPTY_DATASET, "dataset is empty", -1);
  return evaluate_impl(ctx, pop_nodes, pop_conns, P, inputs, targets, batch, fitness_kind, fitness_offset,
                       fitness_out, nullptr);
}

}  // extern "C"

// ---- distance / crossover / rng ---------------------------------------------
namespace fnb {
cudaError_t launch_distance(const double* nodes, const double* conns, int P, const double* rn, const double* rc,
                            int S, int N, int C, double cd, double ch, double* out, void* scratch,
                            size_t scratch_bytes, cudaStream_t st);
size_t distance_scratch_bytes(int S, int N, int C);
cudaError_t launch_crossover(const double* nodes, const double* conns, const int32_t* fit, const int32_t* oth,
                             const uint32_t* keys, int n, int N, int C, double* cn, double* cc, cudaStream_t st);
cudaError_t launch_stream_draws(const uint32_t* keys, int n_keys, int n_draws, int kind, uint64_t n, uint64_t* out,
                                cudaStream_t st);
cudaError_t launch_split_keys(const uint32_t parent[4], uint64_t base, int n, uint32_t* out, cudaStream_t st);
}  // namespace fnb

#include "philox.cuh"

extern "C" {

void fnb_key_seed(uint64_t seed, uint32_t out[4]) {
  const Key4 k = key_from_seed(seed);
  for (int i = 0; i < 4; ++i) out[i] = k.w[i];
}

void fnb_key_split(const uint32_t key[4], uint64_t index, uint32_t out[4]) {
  const Key4 k = key_split(Key4{{key[0], key[1], key[2], key[3]}}, index);
  for (int i = 0; i < 4; ++i) out[i] = k.w[i];
}

int fnb_distance_d(fnb_ctx* ctx, const double* d_nodes, const double* d_conns, int P, const double* d_rep_nodes,
                   const double* d_rep_conns, int S, const fnb_distance_config* cfg, double* d_out, void* stream) {
  if (P <= 0 || S <= 0) return 0;
  if (S > 32) return set_err(ctx, FNB_E_CONFIG_ERROR, "at most 32 representatives per distance call", -1);
  CK(cudaSetDevice(ctx->device));
  const size_t need = distance_scratch_bytes(S, ctx->L.N, ctx->L.C);
  CK(ctx->scratch.ensure(need));
  CK(launch_distance(d_nodes, d_conns, P, d_rep_nodes, d_rep_conns, S, ctx->L.N, ctx->L.C,
                     cfg->compatibility_disjoint, cfg->compatibility_homologous, d_out, ctx->scratch.p,
                     ctx->scratch.cap, static_cast<cudaStream_t>(stream)));
  ctx->launches += kDistanceLaunches;
  return 0;
}

int fnb_crossover_d(fnb_ctx* ctx, const double* d_nodes, const double* d_conns, const int32_t* d_fit,
                    const int32_t* d_other, const uint32_t* d_keys, int n, double* d_child_nodes,
                    double* d_child_conns, void* stream) {
  if (n <= 0) return 0;
  CK(cudaSetDevice(ctx->device));
  CK(launch_crossover(d_nodes, d_conns, d_fit, d_other, d_keys, n, ctx->L.N, ctx->L.C, d_child_nodes,
                      d_child_conns, static_cast<cudaStream_t>(stream)));
  ctx->launches++;
  return 0;
}

int fnb_stream_draws_d(fnb_ctx* ctx, const uint32_t* d_keys, int n_keys, int n_draws, int kind, uint64_t n,
                       uint64_t* d_out, void* stream) {
  if (kind == 2 && n == 0) return set_err(ctx, FNB_E_CONFIG_ERROR, "below(0)", -1);
  CK(cudaSetDevice(ctx->device));
  CK(launch_stream_draws(d_keys, n_keys, n_draws, kind, n, d_out, static_cast<cudaStream_t>(stream)));
  ctx->launches++;
  return 0;
}

int fnb_split_keys_d(fnb_ctx* ctx, const uint32_t key[4], uint64_t base, int n, uint32_t* d_out, void* stream) {
  CK(cudaSetDevice(ctx->device));
  CK(launch_split_keys(key, base, n, d_out, static_cast<cudaStream_t>(stream)));
  ctx->launches++;
  return 0;
}

int fnb_distance(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P, const double* rep_nodes,
                 const double* rep_conns, int S, const fnb_distance_config* cfg, double* out) {
  ctx->err.clear();
  ctx->err_index = -1;
  if (P <= 0 || S <= 0) return 0;
  CK(cudaSetDevice(ctx->device));
  const size_t nb = sizeof(double) * ctx->L.N * kNodeCols, cb = sizeof(double) * ctx->L.C * kConnCols;
  // population and representatives go up in one buffer pair: [pop | reps]
  CK(ctx->nodes.ensure(nb * size_t(P + S)));
  CK(ctx->conns.ensure(cb * size_t(P + S)));
  CK(ctx->out.ensure(sizeof(double) * size_t(P) * S));
  double* dn = static_cast<double*>(ctx->nodes.p);
  double* dc = static_cast<double*>(ctx->conns.p);
  CK(cudaMemcpyAsync(dn, pop_nodes, nb * P, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dc, pop_conns, cb * P, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(dn) + nb * P, rep_nodes, nb * S, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(dc) + cb * P, rep_conns, cb * S, cudaMemcpyHostToDevice, ctx->stream));
  const int st = fnb_distance_d(ctx, dn, dc, P, reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(dn) + nb * P),
                                reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(dc) + cb * P), S, cfg,
                                static_cast<double*>(ctx->out.p), ctx->stream);
  if (st) return st;
  CK(cudaMemcpyAsync(out, ctx->out.p, sizeof(double) * size_t(P) * S, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int fnb_crossover(fnb_ctx* ctx, const double* fit_nodes, const double* fit_conns, const double* other_nodes,
                  const double* other_conns, int n, const uint32_t* keys, double* child_nodes, double* child_conns) {
  ctx->err.clear();
  ctx->err_index = -1;
  if (n <= 0) return 0;
  CK(cudaSetDevice(ctx->device));
  const size_t nb = sizeof(double) * ctx->L.N * kNodeCols, cb = sizeof(double) * ctx->L.C * kConnCols;
  // parents as one 2n population [fit | other]; children after them
  CK(ctx->nodes.ensure(nb * size_t(3 * n)));
  CK(ctx->conns.ensure(cb * size_t(3 * n)));
  CK(ctx->misc.ensure(sizeof(int32_t) * 2 * size_t(n) + sizeof(uint32_t) * 4 * size_t(n) + 64));
  uint8_t* dn = static_cast<uint8_t*>(ctx->nodes.p);
  uint8_t* dc = static_cast<uint8_t*>(ctx->conns.p);
  CK(cudaMemcpyAsync(dn, fit_nodes, nb * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dn + nb * n, other_nodes, nb * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dc, fit_conns, cb * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dc + cb * n, other_conns, cb * n, cudaMemcpyHostToDevice, ctx->stream));
  std::vector<int32_t> idx(2 * size_t(n));
  for (int i = 0; i < n; ++i) { idx[size_t(i)] = i; idx[size_t(n + i)] = n + i; }
  int32_t* d_idx = static_cast<int32_t*>(ctx->misc.p);
  uint32_t* d_keys = reinterpret_cast<uint32_t*>(d_idx + 2 * n);
  CK(cudaMemcpyAsync(d_idx, idx.data(), sizeof(int32_t) * 2 * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(d_keys, keys, sizeof(uint32_t) * 4 * n, cudaMemcpyHostToDevice, ctx->stream));
  const int st = fnb_crossover_d(ctx, reinterpret_cast<double*>(dn), reinterpret_cast<double*>(dc), d_idx,
                                 d_idx + n, d_keys, n, reinterpret_cast<double*>(dn + 2 * nb * n),
                                 reinterpret_cast<double*>(dc + 2 * cb * n), ctx->stream);
  if (st) return st;
  CK(cudaMemcpyAsync(child_nodes, dn + 2 * nb * n, nb * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(child_conns, dc + 2 * cb * n, cb * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

}  // extern "C"

// ---- mutation -----------------------------------------------------------------
namespace fnb {
size_t mutate_scratch_bytes(int n, int N, int C);
cudaError_t launch_mutate(double* nodes, double* conns, const uint32_t* keys, int n, const uint8_t* active,
                          const fnb_mutation_config* m, const DevShape& sh, int* d_next_key, int* d_status,
                          void* scratch, size_t scratch_bytes, int* d_new_key_out, cudaStream_t st,
                          long long* launches);
cudaError_t launch_mutate_plan(const double* nodes, const double* conns, const int32_t* src, const uint32_t* keys,
                               int n, const uint8_t* active, const fnb_mutation_config* m, const DevShape& sh,
                               int* d_next_key, void* scratch, size_t scratch_bytes, int* d_new_key_out,
                               cudaStream_t st, long long* launches);
cudaError_t launch_mutate_apply(double* nodes, double* conns, const uint32_t* keys, int n, int lo, int hi,
                                const uint8_t* active, const fnb_mutation_config* m, const DevShape& sh,
                                int* d_status, void* scratch, size_t scratch_bytes, const int* d_new_key,
                                cudaStream_t st, long long* launches);
void mutate_scratch_views(void* scratch, int n, unsigned long long** pair, int** flag, int** newk);
}  // namespace fnb

extern "C" {

int fnb_mutate_d(fnb_ctx* ctx, double* d_nodes, double* d_conns, int P, const uint32_t* d_keys,
                 const uint8_t* d_active, const fnb_mutation_config* cfg, int* d_next_key, int* d_status,
                 int* d_new_key, void* stream) {
  if (P <= 0) return 0;
  CK(cudaSetDevice(ctx->device));
  CK(ctx->scratch.ensure(mutate_scratch_bytes(P, ctx->L.N, ctx->L.C)));
  CK(launch_mutate(d_nodes, d_conns, d_keys, P, d_active, cfg, ctx->sh, d_next_key, d_status, ctx->scratch.p,
                   ctx->scratch.cap, d_new_key, static_cast<cudaStream_t>(stream), &ctx->launches));
  return 0;
}

int fnb_mutate(fnb_ctx* ctx, double* pop_nodes, double* pop_conns, int P, const uint32_t* keys,
               const fnb_mutation_config* cfg, int* next_key) {
  ctx->err.clear();
  ctx->err_index = -1;
  if (P <= 0) return 0;
  CK(cudaSetDevice(ctx->device));
  const size_t nb = sizeof(double) * ctx->L.N * kNodeCols * size_t(P);
  const size_t cb = sizeof(double) * ctx->L.C * kConnCols * size_t(P);
  CK(ctx->nodes.ensure(nb));
  CK(ctx->conns.ensure(cb));
  // misc: keys [4P] | status [P] | new_key [P] | next_key [2]
  CK(ctx->misc.ensure(sizeof(uint32_t) * 4 * size_t(P) + sizeof(int) * (2 * size_t(P) + 2) + 64));
  uint32_t* d_keys = static_cast<uint32_t*>(ctx->misc.p);
  int* d_status = reinterpret_cast<int*>(d_keys + 4 * size_t(P));
  int* d_newk = d_status + P;
  int* d_nk = d_newk + P;
  const int nk2[2] = {*next_key, 0};
  CK(cudaMemcpyAsync(ctx->nodes.p, pop_nodes, nb, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->conns.p, pop_conns, cb, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(d_keys, keys, sizeof(uint32_t) * 4 * size_t(P), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(d_nk, nk2, sizeof(nk2), cudaMemcpyHostToDevice, ctx->stream));
  int st = fnb_mutate_d(ctx, static_cast<double*>(ctx->nodes.p), static_cast<double*>(ctx->conns.p), P, d_keys,
                        nullptr, cfg, d_nk, d_status, d_newk, ctx->stream);
  if (st) return st;
  std::vector<int> status(static_cast<size_t>(P)), newk(static_cast<size_t>(P));
  CK(cudaMemcpyAsync(status.data(), d_status, sizeof(int) * P, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(newk.data(), d_newk, sizeof(int) * P, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  int bad = -1;
  for (int i = 0; i < P; ++i)
    if (status[size_t(i)]) { bad = i; break; }
  const int done = bad < 0 ? P : bad;  // genomes [0, done) keep their mutation
  const size_t nrow = size_t(ctx->L.N) * kNodeCols, crow = size_t(ctx->L.C) * kConnCols;
  if (done > 0) {
    CK(cudaMemcpyAsync(pop_nodes, ctx->nodes.p, sizeof(double) * nrow * done, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(pop_conns, ctx->conns.p, sizeof(double) * crow * done, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  // table state after slots [0, done] (the failing slot assigned before throwing)
  int nk = *next_key;
  for (int i = 0; i <= (bad < 0 ? P - 1 : bad); ++i)
    if (newk[size_t(i)] >= 0) nk = std::max(nk, newk[size_t(i)] + 1);
  *next_key = nk;
  if (bad >= 0) {
    const int code = status[size_t(bad)] - 1;
    return set_err(ctx, code, code == FNB_E_DUPLICATE_KEY ? "node key " + std::to_string(newk[size_t(bad)])
                                                           : std::string("no free node row"),
                   bad);
  }
  return 0;
}

// mutate() of P genomes in slot order against the CALLER's InnovationTable
// (ops.hpp:145-175, 363-374): the node-split plans (split(0), a pure function
// of each genome) run on the device, the table's get_or_assign is replayed on
// the host in slot order through `assign`, and the keys it hands out drive the
// device apply.  add_node's duplicate-key check (ops.hpp:19-23) is the only
// way a slot can fail; it is tested on the host right after the slot's
// get_or_assign, so the table sees exactly the calls the sequential loop makes
// before it throws.
int fnb_mutate_table(fnb_ctx* ctx, double* pop_nodes, double* pop_conns, int P, const uint32_t* keys,
                     const fnb_mutation_config* cfg, fnb_innovation_fn assign, void* user, int32_t* splits) {
  ctx->err.clear();
  ctx->err_index = -1;
  if (P <= 0) return 0;
  if (!assign) return set_err(ctx, FNB_E_CONFIG_ERROR, "no innovation callback", -1);
  CK(cudaSetDevice(ctx->device));
  const int N = ctx->L.N;
  const size_t nrow = size_t(N) * kNodeCols, crow = size_t(ctx->L.C) * kConnCols;
  const size_t nb = sizeof(double) * nrow * size_t(P), cb = sizeof(double) * crow * size_t(P);
  CK(ctx->nodes.ensure(nb));
  CK(ctx->conns.ensure(cb));
  CK(ctx->scratch.ensure(mutate_scratch_bytes(P, ctx->L.N, ctx->L.C)));
  CK(ctx->misc.ensure(sizeof(uint32_t) * 4 * size_t(P) + sizeof(int) * (size_t(P) + 2) + 64));
  uint32_t* d_keys = static_cast<uint32_t*>(ctx->misc.p);
  int* d_status = reinterpret_cast<int*>(d_keys + 4 * size_t(P));
  int* d_nk = d_status + P;
  const int nk2[2] = {0, 0};
  cudaStream_t st = ctx->stream;
  CK(cudaMemcpyAsync(ctx->nodes.p, pop_nodes, nb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->conns.p, pop_conns, cb, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_keys, keys, sizeof(uint32_t) * 4 * size_t(P), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_nk, nk2, sizeof(nk2), cudaMemcpyHostToDevice, st));
  double* dn = static_cast<double*>(ctx->nodes.p);
  double* dc = static_cast<double*>(ctx->conns.p);
  CK(launch_mutate_plan(dn, dc, nullptr, d_keys, P, nullptr, cfg, ctx->sh, d_nk, ctx->scratch.p, ctx->scratch.cap,
                        nullptr, st, &ctx->launches));
  unsigned long long* d_pair;
  int *d_flag, *d_newk;
  mutate_scratch_views(ctx->scratch.p, P, &d_pair, &d_flag, &d_newk);
  std::vector<unsigned long long> pair(static_cast<size_t>(P));
  std::vector<int> flag(static_cast<size_t>(P)), newk(static_cast<size_t>(P), -1);
  CK(cudaMemcpyAsync(pair.data(), d_pair, sizeof(unsigned long long) * P, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(flag.data(), d_flag, sizeof(int) * P, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int bad = -1;
  for (int c = 0; c < P && bad < 0; ++c) {
    int in_key = 0, out_key = 0;
    if (flag[size_t(c)]) {
      in_key = int(uint32_t(pair[size_t(c)] >> 32));
      out_key = int(uint32_t(pair[size_t(c)]));
      const int k = assign(user, in_key, out_key);
      newk[size_t(c)] = k;
      const double* g = pop_nodes + size_t(c) * nrow;
      for (int r = 0; r < N; ++r)
        if (!std::isnan(g[size_t(r) * kNodeCols]) && int(g[size_t(r) * kNodeCols]) == k) { bad = c; break; }
    }
    if (splits) {
      splits[3 * size_t(c)] = flag[size_t(c)] ? in_key : -1;
      splits[3 * size_t(c) + 1] = flag[size_t(c)] ? out_key : -1;
      splits[3 * size_t(c) + 2] = newk[size_t(c)];
    }
  }
  if (splits)
    for (int c = bad < 0 ? P : bad + 1; c < P; ++c)
      splits[3 * size_t(c)] = splits[3 * size_t(c) + 1] = splits[3 * size_t(c) + 2] = -1;
  const int done = bad < 0 ? P : bad;  // genomes [0, done) are mutated, the rest untouched
  if (done > 0) {
    CK(cudaMemcpyAsync(d_newk, newk.data(), sizeof(int) * size_t(done), cudaMemcpyHostToDevice, st));
    CK(launch_mutate_apply(dn, dc, d_keys, P, 0, done, nullptr, cfg, ctx->sh, d_status, ctx->scratch.p,
                           ctx->scratch.cap, d_newk, st, &ctx->launches));
    std::vector<int> status(static_cast<size_t>(done));
    CK(cudaMemcpyAsync(status.data(), d_status, sizeof(int) * size_t(done), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(pop_nodes, dn, sizeof(double) * nrow * size_t(done), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(pop_conns, dc, sizeof(double) * crow * size_t(done), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int c = 0; c < done; ++c)  // the plan guarantees the rows add_node / add_conn need
      if (status[size_t(c)]) return set_err(ctx, status[size_t(c)] - 1, "mutation failed", c);
  }
  if (bad >= 0) return set_err(ctx, FNB_E_DUPLICATE_KEY, "node key " + std::to_string(newk[size_t(bad)]), bad);
  return 0;
}

}  // extern "C"
