// hyper.cu -- BASELINE config 4: HyperNEAT.  The CPPN population (K1 + K2,
// the same transform and forward as every other config) is queried at the
// substrate's connection coordinates; k_hyper_rollout turns each CPPN's
// outputs into the policy weights of a 27-obs / 8-act substrate and runs the
// synthetic linear-dynamics rollout, one warp per policy.  Semantics:
// DESIGN.md section 9 (restated in FP64 by oracle/hyperneat.c).
//
// The rollout is latency-bound, not bandwidth-bound: see k_hyper_rollout.
#include <algorithm>

#include "fnb_common.cuh"

namespace fnb {

constexpr int kHyperMax = 32;     // n_obs + 1 <= 32 substrate inputs (bias included), n_act <= 32
constexpr int kHyperWarps = 4;

struct HyperParams {
  int n_obs, n_act, steps;
  double thr, wmax;
  float act_cost;
};

// Substrate query rows [(n_obs+1)*n_act][5] (q = j*(n_obs+1) + i).
__global__ void k_hyper_queries(HyperParams hp, float* X) {
  const int ni = hp.n_obs + 1;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ni * hp.n_act) return;
  const int j = q / ni, i = q % ni;
  float* r = X + 5 * size_t(q);
  r[0] = float(-1.0 + 2.0 * i / hp.n_obs);
  r[1] = -1.0f;
  r[2] = float(-1.0 + 2.0 * j / (hp.n_act > 1 ? hp.n_act - 1 : 1));
  r[3] = 1.0f;
  r[4] = 1.0f;
}

// weight = clamp(y, -1, 1) thresholded and rescaled to [-max_weight, max_weight]
__device__ __forceinline__ float hyper_weight(double y, double thr, double wmax) {
  const double v = fmin(1.0, fmax(-1.0, y));
  const double m = fabs(v);
  if (m < thr) return 0.0f;
  const double w = (m - thr) / (1.0 - thr) * wmax;
  return float(v < 0.0 ? -w : w);
}

// One warp per policy.  Policy: lane l computes part (l % G) of output
// j = l / G (G lanes per output, a chunk of CH = 32 / G inputs each, weights in
// registers) and a shfl_xor tree over the G lanes finishes the dot product.
// Dynamics: lane i < n_obs holds A[i] and B[i] in registers.  s (with the
// constant bias input s[n_obs] = 1) and a live in per-warp shared memory
// and are read with broadcast LDS.128.  Each lane sums its reward terms over
// the steps in FP64; one shfl_xor tree combines them at the end.
template <int G>
__global__ void __launch_bounds__(kHyperWarps * 32, G == 4 ? 7 : 3)
k_hyper_rollout(const double* __restrict__ cppn_out, int P, HyperParams hp, const float* __restrict__ A,
                const float* __restrict__ B, const float* __restrict__ s0, double* __restrict__ fitness,
                float* __restrict__ w_out) {
  constexpr int CH = 32 / G;          // inputs per lane of the policy dot product
  constexpr int NA = 32 / G;          // max outputs
  __shared__ __align__(16) float sS[kHyperWarps][kHyperMax];
  __shared__ __align__(16) float sA[kHyperWarps][kHyperMax];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int no = hp.n_obs, na = hp.n_act, ni = no + 1, Q = ni * na;
  const int g = blockIdx.x * kHyperWarps + warp;
  if (g >= P) return;
  const double* y = cppn_out + size_t(g) * Q;
  // policy weights: output j = lane / G, inputs [part * CH, part * CH + CH)
  const int j = lane / G, part = lane % G, i0 = part * CH;
  float wp[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int i = i0 + k;
    float w = 0.0f;
    if (j < na && i < ni) {
      w = hyper_weight(y[j * ni + i], hp.thr, hp.wmax);
      if (w_out) w_out[size_t(g) * Q + j * ni + i] = w;
    }
    wp[k] = w;
  }
  // dynamics rows
  float ar[kHyperMax], br[NA];
#pragma unroll
  for (int k = 0; k < kHyperMax; ++k) ar[k] = (lane < no && k < no) ? A[lane * no + k] : 0.0f;
#pragma unroll
  for (int k = 0; k < NA; ++k) br[k] = (lane < no && k < na) ? B[lane * na + k] : 0.0f;
  float* s = sS[warp];
  float* a = sA[warp];
  s[lane] = lane < no ? s0[lane] : (lane == no ? 1.0f : 0.0f);  // s[n_obs] = the bias input
  a[lane] = 0.0f;
  const float inv_obs = 1.0f / float(no), cost = hp.act_cost / float(na);
  const bool owner = part == 0 && j < na;  // the lane that publishes a_j
  double acc = 0.0;  // this lane's reward terms over the steps
  __syncwarp();
  for (int t = 0; t < hp.steps; ++t) {
    // policy: a_j = tanh(W[j] . [s, 1])
    float z0 = 0.0f, z1 = 0.0f;
#pragma unroll
    for (int k = 0; k < CH; k += 4) {
      const float4 sv = *reinterpret_cast<const float4*>(s + i0 + k);
      z0 = fmaf(wp[k], sv.x, z0);
      z1 = fmaf(wp[k + 1], sv.y, z1);
      z0 = fmaf(wp[k + 2], sv.z, z0);
      z1 = fmaf(wp[k + 3], sv.w, z1);
    }
    float z = z0 + z1;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    const float aj = tanhf(z);
    if (owner) a[j] = aj;
    __syncwarp();
    // dynamics: s'_i = A[i] . s + B[i] . a
    float v0 = 0.0f, v1 = 0.0f, v2 = 0.0f, v3 = 0.0f;
#pragma unroll
    for (int k = 0; k < kHyperMax; k += 4) {
      const float4 sv = *reinterpret_cast<const float4*>(s + k);
      v0 = fmaf(ar[k], sv.x, v0);  // ar[k >= n_obs] = 0 (s[n_obs] is the bias 1)
      v1 = fmaf(ar[k + 1], sv.y, v1);
      v2 = fmaf(ar[k + 2], sv.z, v2);
      v3 = fmaf(ar[k + 3], sv.w, v3);
    }
#pragma unroll
    for (int k = 0; k < NA; k += 4) {
      const float4 av = *reinterpret_cast<const float4*>(a + k);
      v0 = fmaf(br[k], av.x, v0);
      v1 = fmaf(br[k + 1], av.y, v1);
      v2 = fmaf(br[k + 2], av.z, v2);
      v3 = fmaf(br[k + 3], av.w, v3);
    }
    const float v = (v0 + v1) + (v2 + v3);
    __syncwarp();
    if (lane < no) s[lane] = v;
    // reward terms: -(sum s'^2)/n_obs - act_cost (sum a^2)/n_act
    acc -= double((lane < no ? v * v * inv_obs : 0.0f) + (owner ? aj * aj * cost : 0.0f));
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) fitness[g] = acc / hp.steps;
}

cudaError_t launch_hyper_queries(const HyperParams& hp, float* X, cudaStream_t st) {
  const int Q = (hp.n_obs + 1) * hp.n_act;
  k_hyper_queries<<<(Q + 127) / 128, 128, 0, st>>>(hp, X);
  return cudaGetLastError();
}

cudaError_t launch_hyper_rollout(const double* cppn_out, int P, const HyperParams& hp, const float* A,
                                 const float* B, const float* s0, double* fitness, float* w_out, cudaStream_t st) {
  const int grid = (P + kHyperWarps - 1) / kHyperWarps, block = kHyperWarps * 32;
  if (hp.n_act <= 8)
    k_hyper_rollout<4><<<grid, block, 0, st>>>(cppn_out, P, hp, A, B, s0, fitness, w_out);
  else if (hp.n_act <= 16)
    k_hyper_rollout<2><<<grid, block, 0, st>>>(cppn_out, P, hp, A, B, s0, fitness, w_out);
  else
    k_hyper_rollout<1><<<grid, block, 0, st>>>(cppn_out, P, hp, A, B, s0, fitness, w_out);
  return cudaGetLastError();
}

}  // namespace fnb

// ---- C ABI (include/flatneat_b200.h) -------------------------------------------
#include <cstring>
#include <string>

#include "ctx_internal.cuh"

using namespace fnb;

static int hyper_params(fnb_ctx* ctx, const fnb_hyper_config* c, HyperParams* hp) {
  if (!c) return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "hyper config required", -1);
  if (ctx->L.I != 5 || ctx->L.O != 1)
    return fnb_set_error(ctx, FNB_E_SHAPE_MISMATCH, "HyperNEAT CPPNs take 5 inputs (x1, y1, x2, y2, bias) and 1 output",
                         -1);
  if (c->num_obs < 1 || c->num_obs > kHyperMax - 1 || c->num_act < 1 || c->num_act > kHyperMax || c->steps < 1 ||
      !(c->weight_threshold >= 0.0 && c->weight_threshold < 1.0) || !(c->max_weight > 0.0) ||
      !(c->act_cost >= 0.0))
    return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "hyper config out of range (num_obs <= 31, num_act <= 32)", -1);
  *hp = HyperParams{c->num_obs, c->num_act, c->steps, c->weight_threshold, c->max_weight, float(c->act_cost)};
  return 0;
}

#define HCK(expr)                                                  \
  do {                                                             \
    cudaError_t e_ = (expr);                                       \
    if (e_ != cudaSuccess) return fnb_cuda_error(ctx, e_, #expr);  \
  } while (0)

extern "C" {

int fnb_hyper_evaluate_d(fnb_ctx* ctx, const void* d_nets, int P, const fnb_hyper_config* cfg, const float* d_A,
                         const float* d_B, const float* d_s0, double* d_fitness, float* d_weights, void* stream) {
  HyperParams hp;
  if (int st = hyper_params(ctx, cfg, &hp)) return st;
  if (P <= 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HCK(cudaSetDevice(ctx->device));
  const int Q = (hp.n_obs + 1) * hp.n_act;
  const size_t xb = (size_t(Q) * 5 * sizeof(float) + 255) & ~size_t(255);
  HCK(ctx->hyper.ensure(xb + size_t(P) * Q * sizeof(double)));
  float* X = static_cast<float*>(ctx->hyper.p);
  double* out = reinterpret_cast<double*>(static_cast<uint8_t*>(ctx->hyper.p) + xb);
  HCK(launch_hyper_queries(hp, X, s));
  ctx->launches++;
  // the CPPNs at every substrate connection (K2, outputs only)
  if (int st = fnb_forward_d(ctx, d_nets, P, X, nullptr, Q, FNB_FIT_NONE, 0.0, nullptr, out, stream)) return st;
  HCK(launch_hyper_rollout(out, P, hp, d_A, d_B, d_s0, d_fitness, d_weights, s));
  ctx->launches++;
  return 0;
}

int fnb_hyper_evaluate(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P,
                       const fnb_hyper_config* cfg, const double* A, const double* B, const double* s0,
                       double* fitness_out, float* weights_out) {
  ctx->err.clear();
  ctx->err_index = -1;
  HyperParams hp;
  if (int st = hyper_params(ctx, cfg, &hp)) return st;
  if (P <= 0) return 0;
  HCK(cudaSetDevice(ctx->device));
  const int no = hp.n_obs, na = hp.n_act, Q = (no + 1) * na;
  const size_t nb = sizeof(double) * size_t(P) * ctx->L.N * kNodeCols;
  const size_t cb = sizeof(double) * size_t(P) * ctx->L.C * kConnCols;
  HCK(ctx->nodes.ensure(nb));
  HCK(ctx->conns.ensure(cb));
  HCK(ctx->nets.ensure(ctx->L.bytes * size_t(P)));
  HCK(cudaMemcpyAsync(ctx->nodes.p, pop_nodes, nb, cudaMemcpyHostToDevice, ctx->stream));
  HCK(cudaMemcpyAsync(ctx->conns.p, pop_conns, cb, cudaMemcpyHostToDevice, ctx->stream));
  int st = fnb_transform_d(ctx, static_cast<double*>(ctx->nodes.p), static_cast<double*>(ctx->conns.p), P,
                           ctx->nets.p, ctx->stream);
  if (!st)
    st = fnb_check_nets_d(ctx, static_cast<double*>(ctx->nodes.p), static_cast<double*>(ctx->conns.p), ctx->nets.p,
                          P, ctx->stream);
  if (st) return st;
  // dynamics (FP32 on the device), fitness and optional weights
  const size_t na_f = size_t(no) * no + size_t(no) * na + no;
  std::string tmp(sizeof(float) * na_f, '\0');
  float* h = reinterpret_cast<float*>(&tmp[0]);
  for (int i = 0; i < no * no; ++i) h[i] = float(A[i]);
  for (int i = 0; i < no * na; ++i) h[no * no + i] = float(B[i]);
  for (int i = 0; i < no; ++i) h[no * no + no * na + i] = float(s0[i]);
  HCK(ctx->misc.ensure(sizeof(float) * na_f + sizeof(double) * size_t(P) + sizeof(float) * size_t(P) * Q + 512));
  float* dA = static_cast<float*>(ctx->misc.p);
  double* dfit = reinterpret_cast<double*>(static_cast<uint8_t*>(ctx->misc.p) + ((sizeof(float) * na_f + 255) & ~size_t(255)));
  float* dw = weights_out ? reinterpret_cast<float*>(dfit + P) : nullptr;
  HCK(cudaMemcpyAsync(dA, h, sizeof(float) * na_f, cudaMemcpyHostToDevice, ctx->stream));
  st = fnb_hyper_evaluate_d(ctx, ctx->nets.p, P, cfg, dA, dA + no * no, dA + no * no + no * na, dfit, dw,
                            ctx->stream);
  if (st) return st;
  if (fitness_out) HCK(cudaMemcpyAsync(fitness_out, dfit, sizeof(double) * P, cudaMemcpyDeviceToHost, ctx->stream));
  if (weights_out)
    HCK(cudaMemcpyAsync(weights_out, dw, sizeof(float) * size_t(P) * Q, cudaMemcpyDeviceToHost, ctx->stream));
  HCK(cudaStreamSynchronize(ctx->stream));
  return 0;
}

}  // extern "C"
