// forward.cu -- K2: population x sample-batch forward with fused fitness
// (forward_into / batch_forward, network.hpp:238-330; func-fit and XOR
// fitness) on sm_100a CUDA cores.
//
// Mapping: a "group" of T threads evaluates one genome; T = min(256,
// pow2 >= B) so small batches (XOR, B=4) pack many genomes per CTA while
// B >= 256 gives one genome per CTA.  Each thread owns SPT sample columns.
// The genome's op/edge program (K1 output) is staged once into shared
// memory and read as warp-broadcasts; node values live in shared memory as
// v[row][column] so the dynamic source indices of the irregular DAG hit
// conflict-free LDS (consecutive threads = consecutive columns).  A thread
// only ever touches its own columns, so the op loop needs no barriers.
// Arithmetic is FP32 (north star: 1e-5 relative to the FP64 reference);
// the squared-error fitness accumulates in FP64.
#include <algorithm>

#include "fnb_common.cuh"

namespace fnb {

__device__ __forceinline__ float act_apply(int code, float x) {
  switch (code) {  // functions.hpp:17-21
    case FNB_ACT_IDENTITY: return x;
    case FNB_ACT_TANH: return tanhf(x);
    case FNB_ACT_SIGMOID: return 1.0f / (1.0f + expf(-x));
    case FNB_ACT_RELU: return x > 0.0f ? x : 0.0f;
    case FNB_ACT_SIN: return sinf(x);
  }
  return x;
}

struct FwdParams {
  const uint8_t* nets;
  NetLayout L;
  int P;
  const float* X;       // [B][I]
  const float* Y;       // [B][O] or null
  int B;
  int T;                // threads per genome group (power of two)
  int fit_kind;
  double fit_offset;
  double* fitness;      // [P] or null
  double* out;          // [P][B][O] or null
  double* partial;      // [P][chunks] when gridDim.y > 1
  size_t group_smem;    // bytes per group
};

__host__ __device__ inline size_t fwd_group_smem(int N, int C, int I, int O, int T, int spt) {
  size_t b = align16(size_t(N) * sizeof(Op)) + align16(size_t(C) * sizeof(Edge));
  b += align16(size_t(I + O) * sizeof(uint16_t));
  b += align16(size_t(T) * sizeof(double));            // reduction scratch
  b += size_t(N) * size_t(T) * spt * sizeof(float);    // node values
  return align16(b);
}

template <int SPT>
__global__ void __launch_bounds__(256)
k_forward(FwdParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int T = p.T;
  const int groups = blockDim.x / T;
  const int grp = threadIdx.x / T;
  const int j = threadIdx.x % T;
  const int g = blockIdx.x * groups + grp;
  const NetLayout& L = p.L;
  uint8_t* base = smem_raw + size_t(grp) * p.group_smem;
  Op* s_ops = reinterpret_cast<Op*>(base);
  Edge* s_edges = reinterpret_cast<Edge*>(base + align16(size_t(L.N) * sizeof(Op)));
  uint16_t* s_io = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(s_edges) +
                                               align16(size_t(L.C) * sizeof(Edge)));
  double* s_red = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(s_io) +
                                            align16(size_t(L.I + L.O) * sizeof(uint16_t)));
  float* v = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(s_red) + align16(size_t(T) * sizeof(double)));
  const int TC = T * SPT;  // columns per group

  const bool live = g < p.P;
  int n_ops = 0;
  if (live) {
    const uint8_t* net = p.nets + size_t(g) * L.bytes;
    const NetHeader* h = reinterpret_cast<const NetHeader*>(net);
    n_ops = h->n_ops;
    const int n_edges = h->n_edges;
    // stage the program: 16-byte vector copies
    const int4* so = reinterpret_cast<const int4*>(net + L.ops_off);
    int4* dop = reinterpret_cast<int4*>(s_ops);
    for (int i = j; i < n_ops; i += T) dop[i] = so[i];
    const int2* se = reinterpret_cast<const int2*>(net + L.edges_off);
    int2* de = reinterpret_cast<int2*>(s_edges);
    for (int i = j; i < n_edges; i += T) de[i] = se[i];
    const uint16_t* sio = reinterpret_cast<const uint16_t*>(net + L.in_off);
    for (int i = j; i < L.I + L.O; i += T) s_io[i] = sio[i];
  }
  __syncthreads();

  const int I = L.I, O = L.O;
  double err = 0.0;
  // sample tiles assigned to this CTA's y-chunk; dead groups (g >= P) run
  // zero tiles but stay resident for the warp-synchronous reduction below
  const int tiles = (p.B + TC - 1) / TC;
  const int per = (tiles + gridDim.y - 1) / gridDim.y;
  const int t_lo = blockIdx.y * per;
  const int t_hi = live ? min(tiles, t_lo + per) : t_lo;
  for (int tile = t_lo; tile < t_hi; ++tile) {
    int sidx[SPT];
#pragma unroll
    for (int k = 0; k < SPT; ++k) sidx[k] = tile * TC + k * T + j;
    // seed input rows (network.hpp:249-250)
    for (int i = 0; i < I; ++i) {
      float* vr = v + size_t(s_io[i]) * TC;
#pragma unroll
      for (int k = 0; k < SPT; ++k) vr[k * T + j] = sidx[k] < p.B ? p.X[size_t(sidx[k]) * I + i] : 0.0f;
    }
    // ops in topological order (network.hpp:252-264)
    for (int oi = 0; oi < n_ops; ++oi) {
      const Op op = s_ops[oi];
      float acc[SPT];
      if (op.agg == FNB_AGG_SUM || op.agg == FNB_AGG_MEAN) {
#pragma unroll
        for (int k = 0; k < SPT; ++k) acc[k] = 0.0f;
        for (int e = op.e_begin; e < op.e_end; ++e) {
          const Edge ed = s_edges[e];
          const float* vs = v + size_t(ed.src) * TC + j;
#pragma unroll
          for (int k = 0; k < SPT; ++k) acc[k] = fmaf(ed.w, vs[k * T], acc[k]);
        }
        if (op.agg == FNB_AGG_MEAN && op.e_end > op.e_begin) {
          const float n = float(op.e_end - op.e_begin);
#pragma unroll
          for (int k = 0; k < SPT; ++k) acc[k] = acc[k] / n;
        }
      } else if (op.agg == FNB_AGG_PRODUCT) {
#pragma unroll
        for (int k = 0; k < SPT; ++k) acc[k] = 1.0f;
        for (int e = op.e_begin; e < op.e_end; ++e) {
          const Edge ed = s_edges[e];
          const float* vs = v + size_t(ed.src) * TC + j;
#pragma unroll
          for (int k = 0; k < SPT; ++k) acc[k] *= ed.w * vs[k * T];
        }
      } else {  // max; empty fan-in falls back to 0 (network.hpp:258-261)
#pragma unroll
        for (int k = 0; k < SPT; ++k) acc[k] = 0.0f;
        for (int e = op.e_begin; e < op.e_end; ++e) {
          const Edge ed = s_edges[e];
          const float* vs = v + size_t(ed.src) * TC + j;
#pragma unroll
          for (int k = 0; k < SPT; ++k) {
            const float x = ed.w * vs[k * T];
            acc[k] = (e == op.e_begin || x > acc[k]) ? x : acc[k];
          }
        }
      }
      float* vd = v + size_t(op.dst) * TC + j;
#pragma unroll
      for (int k = 0; k < SPT; ++k) vd[k * T] = act_apply(op.act, fmaf(op.resp, acc[k], op.bias));
    }
    // outputs + fitness epilogue
    for (int o = 0; o < O; ++o) {
      const float* vr = v + size_t(s_io[I + o]) * TC + j;
#pragma unroll
      for (int k = 0; k < SPT; ++k) {
        if (sidx[k] >= p.B) continue;
        const float val = vr[k * T];
        if (p.out) p.out[(size_t(g) * p.B + sidx[k]) * O + o] = double(val);
        if (p.fit_kind != FNB_FIT_NONE) {
          const double d = double(p.Y[size_t(sidx[k]) * O + o]) - double(val);
          err += d * d;
        }
      }
    }
  }
  if (p.fit_kind == FNB_FIT_NONE) return;
  // deterministic group reduction: shuffle tree within warps, then ordered
  // sum of warp partials.
  const int width = T < 32 ? T : 32;
  for (int d = width >> 1; d > 0; d >>= 1) err += __shfl_down_sync(0xffffffffu, err, d, width);
  if (T > 32) {
    if ((j & 31) == 0) s_red[j >> 5] = err;
    // all threads of the group are live; sync only this group's warps
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(T));
    if (j == 0) {
      err = 0.0;
      for (int w = 0; w < T / 32; ++w) err += s_red[w];
    }
  }
  if (j == 0 && live) {
    if (gridDim.y > 1) {
      p.partial[size_t(g) * gridDim.y + blockIdx.y] = err;
    } else {
      const double sse = err;
      p.fitness[g] = p.fit_kind == FNB_FIT_NEG_MSE ? -(sse / (double(p.B) * double(O)))
                                                   : p.fit_offset - sse;
    }
  }
}

__global__ void k_fitness_finalize(const double* __restrict__ partial, int chunks, int P, int B, int O,
                                   int fit_kind, double offset, double* __restrict__ fitness) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P) return;
  double sse = 0.0;
  for (int c = 0; c < chunks; ++c) sse += partial[size_t(g) * chunks + c];
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
  int T, groups, chunks, grid_x;
  size_t group_smem, cta_smem;
};

static FwdConfig fwd_config(const NetLayout& L, int P, int B) {
  FwdConfig c{};
  int T = 1;
  while (T < B && T < 256) T <<= 1;
  // keep a CTA's shared memory small enough for >= 2 resident CTAs per SM
  while (T > 32 && fwd_group_smem(L.N, L.C, L.I, L.O, T, 1) * (256 / T) > 100 * 1024) T >>= 1;
  c.T = T;
  c.groups = 256 / T;
  c.group_smem = fwd_group_smem(L.N, L.C, L.I, L.O, T, 1);
  c.cta_smem = c.group_smem * c.groups;
  c.grid_x = (P + c.groups - 1) / c.groups;
  const int tiles = (B + T - 1) / T;
  const int target = 4 * 148;  // >= 4 CTAs per SM before splitting samples
  c.chunks = 1;
  if (c.grid_x < target) c.chunks = std::min(tiles, (target + c.grid_x - 1) / c.grid_x);
  return c;
}

size_t forward_partial_needed(NetLayout L, int P, int B) {
  const FwdConfig c = fwd_config(L, P, B);
  return sizeof(double) * size_t(P) * size_t(c.chunks) + 16;
}

cudaError_t launch_to_float(const double* src, float* dst, size_t n, int* bad, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_to_float<<<int((n + 255) / 256), 256, 0, st>>>(src, dst, n, bad);
  return cudaGetLastError();
}

int launch_forward(const void* nets, NetLayout L, int P, const float* X, const float* Y, int B, int fit_kind,
                   double offset, double* fitness, double* out, double* partial_buf, size_t partial_cap,
                   cudaStream_t st, long long* launches) {
  const FwdConfig c = fwd_config(L, P, B);
  if (c.cta_smem > 227 * 1024) return 1;
  FwdParams p;
  p.nets = static_cast<const uint8_t*>(nets);
  p.L = L;
  p.P = P;
  p.X = X;
  p.Y = Y;
  p.B = B;
  p.T = c.T;
  p.fit_kind = fit_kind;
  p.fit_offset = offset;
  p.fitness = fitness;
  p.out = out;
  p.partial = partial_buf;
  p.group_smem = c.group_smem;
  if (c.chunks > 1 && fit_kind != FNB_FIT_NONE && sizeof(double) * size_t(P) * c.chunks > partial_cap) return 1;
  if (cudaFuncSetAttribute(k_forward<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(c.cta_smem)) !=
      cudaSuccess)
    return 1;
  k_forward<1><<<dim3(c.grid_x, c.chunks), 256, c.cta_smem, st>>>(p);
  if (cudaGetLastError() != cudaSuccess) return 1;
  ++*launches;
  if (c.chunks > 1 && fit_kind != FNB_FIT_NONE) {
    k_fitness_finalize<<<(P + 255) / 256, 256, 0, st>>>(partial_buf, c.chunks, P, B, L.O, fit_kind, offset,
                                                         fitness);
    if (cudaGetLastError() != cudaSuccess) return 1;
    ++*launches;
  }
  return 0;
}

}  // namespace fnb
