// evolve.cu -- the NEAT generation loop on the device (
// PAPER Algorithm 1): initialize_population, speciate, update_stagnation,
// compute_spawn_counts and reproduce, held bit-exact to the frozen CPU
// restatement oracle/evolution.c (the reference ships no code for these
// stages; its rules E1-E5 are listed there and in DESIGN.md).
//
// Everything population-sized is a kernel over genomes or children; the
// species bookkeeping (<= 32 species) runs in single-thread kernels so it
// never leaves the device:
//   speciate   K3 distances to the old representatives -> first match;
//              founding rounds in one cooperative kernel (founder = lowest
//              unassigned index, K3 of the still-unassigned genomes against
//              it, one grid barrier per round); nearest-representative overflow;
//              new representative = member closest to the old one (two-pass
//              atomicMin on (distance bits, index)); empty species dropped.
//   stagnate   per-species max fitness (atomicMax on order-preserving bits),
//              counter update, species_elitism protection, compaction.
//   spawn      fitness mid-ranks from a stable radix sort (CUB), exact
//              integer sums of 2*rank per species, then the clamp / rescale / largest-
//              remainder / elitism arithmetic on one thread.
//   reproduce  members ordered (fitness desc, index asc) from the ranking
//              sort (equal-key groups reversed) and a 6-bit species sort, per-slot parent selection from the split(0) stream,
//              K5 crossover (elites are self-crossovers = exact copies), K6/K7
//              mutation with one slot-ordered innovation table.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <vector>

#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

#include "distance_warp.cuh"
#include "fnb_common.cuh"
#include "glibc_math.cuh"
#include "philox.cuh"

namespace fnb {

namespace cg = cooperative_groups;
constexpr int kMaxSpecies = 32;

struct SpeciesDev {
  int count, next_id, old_count;
  int rcand[kMaxSpecies + 1];  // fused founding rounds: founder of round r (INT_MAX = none)
  int id[kMaxSpecies];
  double best[kMaxSpecies];
  int stag[kMaxSpecies];
  int size[kMaxSpecies];
  int spawn[kMaxSpecies];
  int soff[kMaxSpecies + 1];  // child slot offsets
  int moff[kMaxSpecies + 1];  // member offsets in the sorted member list
  int remap[kMaxSpecies];
  unsigned long long mxbits[kMaxSpecies];
  unsigned long long dmin[kMaxSpecies];
  int argmin[kMaxSpecies];
  long long rsum[kMaxSpecies];
  int cnt[kMaxSpecies];
  int total_spawn;
  int error;
  int generation;    // the step's generation (keys split(1).split(generation)); graph replays read it here
  int first_bad;     // lowest child whose mutation failed (INT_MAX = none)
};

struct NeatCfg {  // == fnb_neat_config
  int pop_size, max_species;
  double threshold;
  int species_elitism, max_stagnation, genome_elitism;
  double survival, spawn_rate;
  int output_activation;
};

__device__ __forceinline__ unsigned long long ordered_bits(double x) {  // monotone in x; -0 == +0
  x = __dadd_rn(x, 0.0);
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_ordered(unsigned long long o) {
  const unsigned long long u = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  return __longlong_as_double((long long)u);
}

// ---- initialize_population (oracle E1) ------------------------
__global__ void k_init_population(double* nodes, double* conns, int P, int N, int C, int I, int O, Key4 init_key,
                                  double bm, double bs, double rm, double rs, double wm, double ws, int default_agg,
                                  int default_act, int out_act) {
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= P) return;
  double* n = nodes + size_t(g) * N * kNodeCols;
  double* c = conns + size_t(g) * C * kConnCols;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  for (int i = lane; i < N * kNodeCols; i += 32) n[i] = nan;
  for (int i = lane; i < C * kConnCols; i += 32) c[i] = nan;
  __syncwarp();
  if (lane != 0) return;
  Stream s(key_split(init_key, uint64_t(g)));
  const int hidden = I + O;
  for (int i = 0; i < I; ++i) {
    double* row = n + i * kNodeCols;
    row[0] = double(i); row[1] = 0.0; row[2] = 1.0; row[3] = double(default_agg); row[4] = double(default_act);
  }
  for (int r = I; r <= hidden; ++r) {
    double* row = n + r * kNodeCols;
    row[0] = double(r);
    const double a0 = s.uniform(), a1 = s.uniform();
    row[1] = glibc::normal_from_uniforms(a0, a1, bm, bs);
    const double b0 = s.uniform(), b1 = s.uniform();
    row[2] = glibc::normal_from_uniforms(b0, b1, rm, rs);
    row[3] = double(default_agg);
    row[4] = double(r < hidden ? out_act : default_act);
  }
  for (int r = 0; r < I + O; ++r) {
    double* row = c + r * kConnCols;
    row[0] = double(r < I ? r : hidden);
    row[1] = double(r < I ? hidden : r);
    row[2] = 1.0;
    const double a0 = s.uniform(), a1 = s.uniform();
    row[3] = glibc::normal_from_uniforms(a0, a1, wm, ws);
  }
}

// copy genome `src` (or *src_dev when src < 0) into dst
__global__ void k_copy_genome(const double* sn, const double* sc, const int* src_dev, int src, double* dn, double* dc,
                              int N, int C) {
  const int s = src >= 0 ? src : *src_dev;
  if (s < 0) return;
  const double* a = sn + size_t(s) * N * kNodeCols;
  const double* b = sc + size_t(s) * C * kConnCols;
  for (int i = threadIdx.x; i < N * kNodeCols; i += blockDim.x) dn[i] = a[i];
  for (int i = threadIdx.x; i < C * kConnCols; i += blockDim.x) dc[i] = b[i];
}

// ---- speciate (oracle E2) -------------------------------------------------------
__global__ void k_spec_begin(SpeciesDev* sd) {
  sd->old_count = sd->count;
  for (int j = 0; j <= kMaxSpecies; ++j) sd->rcand[j] = INT_MAX;
  sd->first_bad = INT_MAX;
  for (int j = 0; j < kMaxSpecies; ++j) {
    sd->dmin[j] = 0x7fffffffffffffffull;  // above every distance bits, and positive as int64 (sharded MIN)
    sd->argmin[j] = INT_MAX;
    sd->size[j] = 0;
  }
}

// Per-genome kernels of the step take a genome range [lo, hi): the whole
// population in one process, a rank's shard in the sharded step.
__global__ void k_assign_first(const double* __restrict__ d, int lo, int hi, int S_old, double th, int* species_of) {
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hi) return;
  int a = -1;
  for (int j = 0; j < S_old; ++j)
    if (d[size_t(i) * S_old + j] < th) { a = j; break; }
  species_of[i] = a;
}

// All founding rounds in one cooperative launch (oracle E2, the rounds of
// founder search, founder commit, K3 against the founder and the join fused):
// round r's founder f is the lowest unassigned genome; it founds species
// j = S_old + r, and every unassigned genome after it whose distance to it is
// below the threshold joins.  Genomes that stay unassigned atomicMin the
// next round's founder, so no separate minimum pass is needed; each CTA
// builds the founder's marker tables in its own shared memory, so the only
// grid-wide barrier is one per round.  Rounds end, grid-uniformly, when no
// genome is left or max_species is reached.  Distances are distance_warp's
// (bit-identical to k_distance).
__global__ void __launch_bounds__(128) k_found_rounds(SpeciesDev* sd, int S_old, int max_species, int* species_of,
                                                      const double* __restrict__ pn, const double* __restrict__ pc,
                                                      double* rep_n, double* rep_c, int P, int N, int C, double th,
                                                      double cd, double ch, int Hn, int Hc) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) uint8_t smem_raw[];
  unsigned long long* nk = reinterpret_cast<unsigned long long*>(smem_raw);
  unsigned long long* ck = nk + Hn;
  double* cw = reinterpret_cast<double*>(ck + Hc);
  int* nr = reinterpret_cast<int*>(cw + Hc);
  int* cr = nr + Hn;
  int* counts = cr + Hc;                                          // 2 ints (+2 pad)
  double* dist_w = reinterpret_cast<double*>(counts + 4);         // one per warp
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* tile = dist_w + warps + size_t(warp) * 33;  // distance_warp scratch (S = 1)
  const int gw = blockIdx.x * warps + warp, nw = gridDim.x * warps;
  const size_t gn = size_t(N) * kNodeCols, gc = size_t(C) * kConnCols;

  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x)
    if (__ldcg(species_of + i) < 0) atomicMin(&sd->rcand[0], i);
  grid.sync();
  for (int r = 0; S_old + r < max_species; ++r) {
    const int f = __ldcg(&sd->rcand[r]);
    if (f == INT_MAX) break;
    const int j = S_old + r;
    const double* fn = pn + size_t(f) * gn;
    const double* fc = pc + size_t(f) * gc;
    if (blockIdx.x == 0) {  // commit the species and its representative
      if (threadIdx.x == 0) {
        sd->count = j + 1;
        sd->id[j] = sd->next_id++;
        sd->best[j] = -INFINITY;
        sd->stag[j] = 0;
        species_of[f] = j;
      }
      for (size_t i = threadIdx.x; i < gn; i += blockDim.x) rep_n[size_t(j) * gn + i] = fn[i];
      for (size_t i = threadIdx.x; i < gc; i += blockDim.x) rep_c[size_t(j) * gc + i] = fc[i];
    }
    rep_table_build(fn, fc, N, C, nk, nr, Hn, ck, cr, cw, Hc, counts);
    const RepTables t{nk, nr, ck, cr, cw, counts, Hn, Hc, nullptr, 0};
    for (int g = gw; g < P; g += nw) {
      if (g <= f || __ldcg(species_of + g) >= 0) continue;  // warp-uniform
      distance_warp(pn + size_t(g) * gn, pc + size_t(g) * gc, fn, fc, 1, t, N, C, cd, ch, tile, dist_w + warp);
      __syncwarp();
      if (lane == 0) {
        if (dist_w[warp] < th) species_of[g] = j;
        else atomicMin(&sd->rcand[r + 1], g);
      }
      __syncwarp();
    }
    grid.sync();
  }
}

// Members by (fitness descending, index ascending) from the ascending stable
// sort (keys desc = ~asc): the equal-key group [lo, hi) of position i moves
// to [P - hi, P - lo), keeping its (index-ascending) order -- replaces a
// second 64-bit radix sort with two binary searches per element.
__global__ void k_desc_from_asc(const unsigned long long* __restrict__ keys, const int* __restrict__ idx, int P,
                                int* __restrict__ out, int* __restrict__ rank2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const unsigned long long k = keys[i];
  int a = 0, b = i;  // lo = first position with key >= k
  while (a < b) {
    const int m = (a + b) >> 1;
    if (keys[m] < k) a = m + 1;
    else b = m;
  }
  const int lo = a;
  a = i + 1;
  b = P;  // hi = first position with key > k
  while (a < b) {
    const int m = (a + b) >> 1;
    if (keys[m] <= k) a = m + 1;
    else b = m;
  }
  out[(P - a) + (i - lo)] = idx[i];
  rank2[i] = lo + a - 1;  // 2 x the mid-rank of position i (oracle E4): the tie group is [lo, a)
}

__global__ void k_nearest(const double* __restrict__ d, int lo, int hi, int stride, const SpeciesDev* sd,
                          int* species_of) {
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hi || species_of[i] >= 0) return;
  int best = 0;
  double bd = 0.0;
  for (int j = 0; j < sd->count; ++j) {
    const double x = d[size_t(i) * stride + j];
    if (j == 0 || x < bd) { bd = x; best = j; }
  }
  species_of[i] = best;
}

__global__ void k_rep_min(const double* __restrict__ d, int lo, int hi, int S_old, const int* species_of,
                          SpeciesDev* sd, int pass) {
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hi) return;
  const int j = species_of[i];
  if (j < 0 || j >= S_old) return;
  const unsigned long long b = (unsigned long long)__double_as_longlong(d[size_t(i) * S_old + j]);  // d >= 0
  if (pass == 0) atomicMin(&sd->dmin[j], b);
  else if (b == sd->dmin[j]) atomicMin(&sd->argmin[j], i);
}

// new representatives of old species: one block per species
__global__ void k_rep_copy(const SpeciesDev* sd, const double* pn, const double* pc, double* rep_n, double* rep_c,
                           int N, int C) {
  const int j = blockIdx.x;
  if (j >= sd->old_count) return;
  const int m = sd->argmin[j];
  if (m == INT_MAX) return;
  for (int i = threadIdx.x; i < N * kNodeCols; i += blockDim.x)
    rep_n[size_t(j) * N * kNodeCols + i] = pn[size_t(m) * N * kNodeCols + i];
  for (int i = threadIdx.x; i < C * kConnCols; i += blockDim.x)
    rep_c[size_t(j) * C * kConnCols + i] = pc[size_t(m) * C * kConnCols + i];
}

// Per-species integer reductions are aggregated per CTA in shared memory
// first (a few species, thousands of genomes: global same-address atomics
// serialise); integer adds and max are order-independent, so no bit moves.
__global__ void k_sizes(const int* species_of, int lo, int hi, SpeciesDev* sd) {
  __shared__ int s_n[kMaxSpecies];
  for (int t = threadIdx.x; t < kMaxSpecies; t += blockDim.x) s_n[t] = 0;
  __syncthreads();
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < hi && species_of[i] >= 0) atomicAdd(&s_n[species_of[i]], 1);
  __syncthreads();
  for (int t = threadIdx.x; t < kMaxSpecies; t += blockDim.x)
    if (s_n[t]) atomicAdd(&sd->size[t], s_n[t]);
}

__global__ void k_mark_nonempty(SpeciesDev* sd) {
  for (int j = 0; j < sd->count; ++j) sd->remap[j] = sd->size[j] > 0 ? 1 : -1;
}

// compaction driven by remap[j] in {1 keep, -1 drop}: rewrites remap to the
// new index and moves every field and representative (new <= old: forward)
__global__ void k_apply_compaction(SpeciesDev* sd, double* rep_n, double* rep_c, int N, int C) {
  __shared__ int S;
  if (threadIdx.x == 0) {
    S = sd->count;
    int k = 0;
    for (int j = 0; j < S; ++j) sd->remap[j] = sd->remap[j] > 0 ? k++ : -1;
  }
  __syncthreads();
  for (int j = 0; j < S; ++j) {
    const int t = sd->remap[j];
    if (t < 0 || t == j) continue;
    for (int i = threadIdx.x; i < N * kNodeCols; i += blockDim.x)
      rep_n[size_t(t) * N * kNodeCols + i] = rep_n[size_t(j) * N * kNodeCols + i];
    for (int i = threadIdx.x; i < C * kConnCols; i += blockDim.x)
      rep_c[size_t(t) * C * kConnCols + i] = rep_c[size_t(j) * C * kConnCols + i];
    __syncthreads();
    if (threadIdx.x == 0) {
      sd->id[t] = sd->id[j];
      sd->best[t] = sd->best[j];
      sd->stag[t] = sd->stag[j];
      sd->size[t] = sd->size[j];
      sd->spawn[t] = sd->spawn[j];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int k = 0;
    for (int j = 0; j < S; ++j) k += sd->remap[j] >= 0;
    sd->count = k;
  }
}

__global__ void k_remap(int* species_of, int lo, int hi, const SpeciesDev* sd) {
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < hi && species_of[i] >= 0) species_of[i] = sd->remap[species_of[i]];
}

// ---- update_stagnation (oracle E3) --------------------------------------------------
__global__ void k_stag_begin(SpeciesDev* sd) {
  for (int j = 0; j < kMaxSpecies; ++j) sd->mxbits[j] = 0ull;
}
__global__ void k_species_max(const double* fitness, const int* species_of, int lo, int hi, SpeciesDev* sd) {
  __shared__ unsigned long long s_mx[kMaxSpecies];
  for (int t = threadIdx.x; t < kMaxSpecies; t += blockDim.x) s_mx[t] = 0ull;
  __syncthreads();
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < hi && species_of[i] >= 0) atomicMax(&s_mx[species_of[i]], ordered_bits(fitness[i]));
  __syncthreads();
  for (int t = threadIdx.x; t < kMaxSpecies; t += blockDim.x)
    if (s_mx[t]) atomicMax(&sd->mxbits[t], s_mx[t]);
}
__global__ void k_stagnation(SpeciesDev* sd, int species_elitism, int max_stagnation) {
  const int S = sd->count;
  if (S <= 0) return;
  double mx[kMaxSpecies];
  for (int j = 0; j < S; ++j) mx[j] = from_ordered(sd->mxbits[j]);
  for (int j = 0; j < S; ++j) {
    if (mx[j] > sd->best[j]) { sd->best[j] = mx[j]; sd->stag[j] = 0; }
    else sd->stag[j] += 1;
  }
  int prot[kMaxSpecies];
  for (int j = 0; j < S; ++j) {
    int better = 0;
    for (int q = 0; q < S; ++q)
      if (mx[q] > mx[j] || (mx[q] == mx[j] && q < j)) ++better;
    prot[j] = better < species_elitism;
  }
  int survivors = 0;
  for (int j = 0; j < S; ++j) survivors += (prot[j] || sd->stag[j] <= max_stagnation);
  if (survivors == 0) {
    int b = 0;
    for (int j = 1; j < S; ++j)
      if (mx[j] > mx[b]) b = j;
    prot[b] = 1;
  }
  for (int j = 0; j < S; ++j) sd->remap[j] = (!prot[j] && sd->stag[j] > max_stagnation) ? -1 : 1;
}
__global__ void k_remap_or_drop(int* species_of, int lo, int hi, const SpeciesDev* sd) {
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < hi && species_of[i] >= 0) species_of[i] = sd->remap[species_of[i]];
}

// ---- compute_spawn_counts (oracle E4) ------------------------------------------------
__global__ void k_fit_keys(const double* fitness, int P, unsigned long long* asc, unsigned long long* desc, int* idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const unsigned long long o = ordered_bits(fitness[i]);
  asc[i] = o;
  desc[i] = ~o;
  idx[i] = i;
}
// mid-ranks (oracle E4): position r of the ascending sort lies in the tie
// group [lo, hi) of its key; 2 * rank = lo + hi - 1 (k_desc_from_asc), an
// exact integer
__global__ void k_rank_sums(const int* __restrict__ rank2, const int* sorted_idx, int P, const int* species_of,
                            int lo, int hi, SpeciesDev* sd) {
  __shared__ unsigned long long s_sum[kMaxSpecies];
  __shared__ int s_cnt[kMaxSpecies];
  for (int t = threadIdx.x; t < kMaxSpecies; t += blockDim.x) {
    s_sum[t] = 0ull;
    s_cnt[t] = 0;
  }
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int gi = r < P ? sorted_idx[r] : -1;
  if (r < P && gi >= lo && gi < hi) {  // this process's genomes; ranks are over the whole population
    const int j = species_of[gi];
    if (j >= 0) {
      atomicAdd(&s_sum[j], (unsigned long long)rank2[r]);
      atomicAdd(&s_cnt[j], 1);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kMaxSpecies; t += blockDim.x)
    if (s_cnt[t]) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&sd->rsum[t]), s_sum[t]);
      atomicAdd(&sd->cnt[t], s_cnt[t]);
    }
}
__global__ void k_spawn_begin(SpeciesDev* sd) {
  for (int j = 0; j < kMaxSpecies; ++j) { sd->rsum[j] = 0; sd->cnt[j] = 0; }
}
__global__ void k_spawn(SpeciesDev* sd, int P, double rate, int genome_elitism) {
  const int S = sd->count;
  double af[kMaxSpecies], nw[kMaxSpecies], frac[kMaxSpecies];
  double total = 0.0;
  for (int j = 0; j < S; ++j) {
    af[j] = __ddiv_rn(double(sd->rsum[j]), __dmul_rn(__dmul_rn(2.0, double(P - 1)), double(sd->cnt[j])));
    total = __dadd_rn(total, af[j]);
  }
  double sum_new = 0.0;
  for (int j = 0; j < S; ++j) {
    const double target = total > 0.0 ? __dmul_rn(__ddiv_rn(af[j], total), double(P)) : __ddiv_rn(double(P), double(S));
    const double old = double(sd->cnt[j]);
    const double md = round(__dmul_rn(rate, old));
    double v = target;
    if (v < __dsub_rn(old, md)) v = __dsub_rn(old, md);
    if (v > __dadd_rn(old, md)) v = __dadd_rn(old, md);
    nw[j] = v;
    sum_new = __dadd_rn(sum_new, v);
  }
  int assigned = 0;
  for (int j = 0; j < S; ++j) {
    const double sc = sum_new > 0.0 ? __ddiv_rn(__dmul_rn(nw[j], double(P)), sum_new) : __ddiv_rn(double(P), double(S));
    const double fl = floor(sc);
    sd->spawn[j] = int(fl);
    frac[j] = __dsub_rn(sc, fl);
    assigned += sd->spawn[j];
  }
  int rem = P - assigned;
  while (rem > 0) {
    int b = -1;
    for (int j = 0; j < S; ++j)
      if (frac[j] >= 0.0 && (b < 0 || frac[j] > frac[b])) b = j;
    if (b < 0) {
      for (int j = 0; j < S && rem > 0; ++j, --rem) sd->spawn[j]++;
      break;
    }
    sd->spawn[b]++;
    frac[b] = -1.0;
    --rem;
  }
  int tot = 0;
  for (int j = 0; j < S; ++j) {
    if (sd->spawn[j] < genome_elitism) sd->spawn[j] = genome_elitism;
    tot += sd->spawn[j];
  }
  while (tot > P) {
    int b = -1;
    for (int j = 0; j < S; ++j)
      if (sd->spawn[j] > genome_elitism && (b < 0 || sd->spawn[j] >= sd->spawn[b])) b = j;
    if (b < 0) break;
    sd->spawn[b]--;
    --tot;
  }
  int so = 0, mo = 0;
  for (int j = 0; j < S; ++j) {
    sd->soff[j] = so;
    sd->moff[j] = mo;
    so += sd->spawn[j];
    mo += sd->cnt[j];
    sd->size[j] = sd->cnt[j];
  }
  sd->soff[S] = so;
  sd->moff[S] = mo;
  sd->total_spawn = so;
  sd->error = so == P ? 0 : 1;
}

// ---- reproduce (oracle E5) -----------------------------------------------------------------
__global__ void k_species_keys(const int* sorted_idx, int P, const int* species_of, int* skey) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P) return;
  const int j = species_of[sorted_idx[r]];
  skey[r] = j < 0 ? kMaxSpecies : j;
}

__global__ void k_gen_advance(SpeciesDev* sd) { ++sd->generation; }

__global__ void k_first_bad(const int* status, int n, SpeciesDev* sd, int base) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && status[i]) atomicMin(&sd->first_bad, base + i);
}

__global__ void k_reproduce_plan(const SpeciesDev* sd, const int* members, const double* fitness, int P, Key4 root1,
                                 int genome_elitism, double survival, int* fit_idx, int* oth_idx, uint32_t* xkeys,
                                 uint32_t* mkeys, uint8_t* active) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P) return;
  const int S = sd->count;
  int j = 0;
  while (j + 1 < S && sd->soff[j + 1] <= c) ++j;
  const int k = c - sd->soff[j];
  const int m = sd->size[j];
  const int* mem = members + sd->moff[j];
  int n_elite = genome_elitism;
  if (n_elite > sd->spawn[j]) n_elite = sd->spawn[j];
  if (n_elite > m) n_elite = m;
  if (k < n_elite) {  // elite: exact copy (self-crossover), not mutated
    fit_idx[c] = oth_idx[c] = mem[k];
    for (int q = 0; q < 4; ++q) { xkeys[4 * c + q] = 0u; mkeys[4 * c + q] = 0u; }
    active[c] = 0;
    return;
  }
  int pool = int(ceil(__dmul_rn(survival, double(m))));
  if (pool < 1) pool = 1;
  if (pool > m) pool = m;
  const Key4 ck = key_split(key_split(root1, uint64_t(sd->generation)), uint64_t(c));
  Stream sel(key_split(ck, 0));
  const uint64_t lim = Stream::below_limit(uint64_t(pool));
  const int a = mem[sel.index_lim(pool, lim)];
  const int b = mem[sel.index_lim(pool, lim)];
  const bool a_fit = fitness[a] > fitness[b] || (fitness[a] == fitness[b] && a <= b);
  fit_idx[c] = a_fit ? a : b;
  oth_idx[c] = a_fit ? b : a;
  const Key4 xk = key_split(ck, 1), mk = key_split(ck, 2);
  for (int q = 0; q < 4; ++q) { xkeys[4 * c + q] = xk.w[q]; mkeys[4 * c + q] = mk.w[q]; }
  active[c] = 1;
}

// Populations up to kCountRankMax: the two stable sorts of the step (fitness
// ranks, then members by species) are a counting rank -- the position of
// item i is #(k_j < k_i) + #(k_j == k_i, j < i), exactly the stable sort's --
// spread over the whole GPU (O(P^2) compares, ~1e8 at pop 10k, a few
// microseconds) and a scatter, instead of a chain of radix-sort kernels.
// Grid: x = blocks of 256 items, y = tiles of 256 keys staged in shared
// memory; a tile wholly before / after a block compares with <= / <, only
// the tile holding the block breaks ties by index.  Partial counts are
// summed with integer atomics (order-independent).
constexpr int kCountRankMax = 16384;
constexpr int kRankItems = 256, kRankTile = 256;

template <typename K>
__global__ void __launch_bounds__(128) k_count_rank(const K* __restrict__ keys, int n, int* __restrict__ rank) {
  __shared__ K sk[kRankTile];
  const int ib = blockIdx.x * kRankItems, j0 = blockIdx.y * kRankTile;
  const int jn = min(kRankTile, n - j0);
  for (int t = threadIdx.x; t < jn; t += blockDim.x) sk[t] = keys[j0 + t];
  __syncthreads();
  const int i0 = ib + threadIdx.x, i1 = i0 + 128;
  const K k0 = i0 < n ? keys[i0] : K(0), k1 = i1 < n ? keys[i1] : K(0);
  int c0 = 0, c1 = 0;
  if (j0 + jn <= ib) {
#pragma unroll 8
    for (int j = 0; j < jn; ++j) {
      const K kj = sk[j];
      c0 += kj <= k0;
      c1 += kj <= k1;
    }
  } else if (j0 >= ib + kRankItems) {
#pragma unroll 8
    for (int j = 0; j < jn; ++j) {
      const K kj = sk[j];
      c0 += kj < k0;
      c1 += kj < k1;
    }
  } else {
    for (int j = 0; j < jn; ++j) {
      const K kj = sk[j];
      const int jj = j0 + j;
      c0 += (kj < k0) | ((kj == k0) & (jj < i0));
      c1 += (kj < k1) | ((kj == k1) & (jj < i1));
    }
  }
  if (i0 < n && c0) atomicAdd(&rank[i0], c0);
  if (i1 < n && c1) atomicAdd(&rank[i1], c1);
}

// out position rank[i] receives item i: its key (when kout) and vals[i] (i when vals is null)
template <typename K>
__global__ void k_rank_scatter(const K* __restrict__ keys, const int* __restrict__ vals, const int* __restrict__ rank,
                               int n, K* __restrict__ kout, int* __restrict__ vout) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = rank[i];
  if (kout) kout[r] = keys[i];
  vout[r] = vals ? vals[i] : i;
}

template <typename K>
cudaError_t launch_count_sort(const K* keys, const int* vals, int n, int* rank, K* kout, int* vout, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(rank, 0, sizeof(int) * size_t(n), st);
  if (e != cudaSuccess) return e;
  const dim3 grid((n + kRankItems - 1) / kRankItems, (n + kRankTile - 1) / kRankTile);
  k_count_rank<K><<<grid, 128, 0, st>>>(keys, n, rank);
  k_rank_scatter<K><<<(n + 255) / 256, 256, 0, st>>>(keys, vals, rank, n, kout, vout);
  return cudaGetLastError();
}

// ---- host-side launchers used by capi.cu ------------------------------------------------------
cudaError_t launch_distance_masked(const double* nodes, const double* conns, int P, const double* rn,
                                   const double* rc, int S, int N, int C, double cd, double ch, double* out,
                                   void* scratch, size_t scratch_bytes, const int* only_unassigned,
                                   const int* after_founder, cudaStream_t st);
size_t distance_scratch_bytes(int S, int N, int C);
cudaError_t launch_crossover(const double* nodes, const double* conns, const int32_t* fit, const int32_t* oth,
                             const uint32_t* keys, int n, int N, int C, double* cn, double* cc, cudaStream_t st);
size_t mutate_scratch_bytes(int n, int N, int C);
cudaError_t launch_mutate_plan(const double* nodes, const double* conns, const int32_t* src, const uint32_t* keys,
                               int n, const uint8_t* active, const fnb_mutation_config* m, const DevShape& sh,
                               int* d_next_key, void* scratch, size_t scratch_bytes, int* d_new_key_out,
                               cudaStream_t st, long long* launches);
cudaError_t launch_mutate_apply(double* nodes, double* conns, const uint32_t* keys, int n, int lo, int hi,
                                const uint8_t* active, const fnb_mutation_config* m, const DevShape& sh,
                                int* d_status, void* scratch, size_t scratch_bytes, const int* d_new_key,
                                cudaStream_t st, long long* launches);


// ---- the step sharded over ranks (distributed.py ShardedEvolution) ----------------
// Rank r owns genomes [lo, hi) of full-size buffers (global genome indices
// everywhere).  The kernels below are the rank-local parts of speciate /
// stagnation / spawn / reproduce; the collectives between them (all-reduce
// MIN / MAX / SUM of exact integers or order-preserving bits, broadcast of a
// founder, all-gathers of fitness, species ids and parent genomes) run in the
// caller, so the result is the one-process step bit for bit.
__global__ void k_set_int(int* p, int v) { *p = v; }

__global__ void k_min_unassigned(const int* species_of, int lo, int hi, int* out) {
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  const bool u = i < hi && species_of[i] < 0;
  const unsigned b = __ballot_sync(0xffffffffu, u);
  if (b && (threadIdx.x & 31) == __ffs(b) - 1) atomicMin(out, i);
}

// the founder's owner: representative slot j <- genome f, f joins species j
__global__ void k_found_copy(const double* pn, const double* pc, int f, int j, double* rep_n, double* rep_c,
                             int* species_of, int N, int C) {
  const size_t gn = size_t(N) * kNodeCols, gc = size_t(C) * kConnCols;
  for (size_t i = threadIdx.x; i < gn; i += blockDim.x) rep_n[size_t(j) * gn + i] = pn[size_t(f) * gn + i];
  for (size_t i = threadIdx.x; i < gc; i += blockDim.x) rep_c[size_t(j) * gc + i] = pc[size_t(f) * gc + i];
  if (threadIdx.x == 0) species_of[f] = j;
}

// every rank: species j exists (oracle E2 founding), as k_found_rounds commits it
__global__ void k_found_commit(SpeciesDev* sd, int j) {
  sd->count = j + 1;
  sd->id[j] = sd->next_id++;
  sd->best[j] = -INFINITY;
  sd->stag[j] = 0;
}

__global__ void k_join(const double* __restrict__ d, int lo, int hi, double th, int j, int* species_of) {
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < hi && species_of[i] < 0 && d[i] < th) species_of[i] = j;
}

// new representative candidates: slot j holds genome argmin[j]'s bits on
// its owner and zeros elsewhere, so an integer SUM over ranks is a gather
__global__ void k_rep_stage(const SpeciesDev* sd, const double* pn, const double* pc, int lo, int hi,
                            unsigned long long* stage, int N, int C) {
  const int j = blockIdx.x;
  const size_t gn = size_t(N) * kNodeCols, gc = size_t(C) * kConnCols;
  const int m = sd->argmin[j];
  const bool mine = m != INT_MAX && m >= lo && m < hi;
  unsigned long long* dst = stage + size_t(j) * (gn + gc);
  const unsigned long long* a = reinterpret_cast<const unsigned long long*>(pn) + (mine ? size_t(m) * gn : 0);
  const unsigned long long* b = reinterpret_cast<const unsigned long long*>(pc) + (mine ? size_t(m) * gc : 0);
  for (size_t i = threadIdx.x; i < gn; i += blockDim.x) dst[i] = mine ? a[i] : 0ull;
  for (size_t i = threadIdx.x; i < gc; i += blockDim.x) dst[gn + i] = mine ? b[i] : 0ull;
}
__global__ void k_rep_commit(const SpeciesDev* sd, const unsigned long long* stage, double* rep_n, double* rep_c,
                             int N, int C) {
  const int j = blockIdx.x;
  if (j >= sd->old_count || sd->argmin[j] == INT_MAX) return;
  const size_t gn = size_t(N) * kNodeCols, gc = size_t(C) * kConnCols;
  const unsigned long long* src = stage + size_t(j) * (gn + gc);
  unsigned long long* rn = reinterpret_cast<unsigned long long*>(rep_n) + size_t(j) * gn;
  unsigned long long* rc = reinterpret_cast<unsigned long long*>(rep_c) + size_t(j) * gc;
  for (size_t i = threadIdx.x; i < gn; i += blockDim.x) rn[i] = src[i];
  for (size_t i = threadIdx.x; i < gc; i += blockDim.x) rc[i] = src[gn + i];
}

// parents: genomes some slot reads (elites are self-crossovers)
__global__ void k_need(const int* fit_idx, const int* oth_idx, int P, int* need) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < P) {
    need[fit_idx[c]] = 1;
    need[oth_idx[c]] = 1;
  }
}
// exclusive scan of need[P] into prefix[P + 1] (one CTA, contiguous runs per thread)
__global__ void __launch_bounds__(1024) k_scan_need(const int* need, int P, int* prefix) {
  __shared__ int warp_sums[32];
  const int t = threadIdx.x, nt = blockDim.x;
  const int per = (P + nt - 1) / nt;
  const int lo = min(P, t * per), hi = min(P, lo + per);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += need[i];
  const int lane = t & 31, w = t >> 5;
  int incl = cnt;
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  if (lane == 31) warp_sums[w] = incl;
  __syncthreads();
  if (w == 0) {
    int v = lane < (nt >> 5) ? warp_sums[lane] : 0;
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= d) v += u;
    }
    warp_sums[lane] = v;
  }
  __syncthreads();
  int run = (w > 0 ? warp_sums[w - 1] : 0) + incl - cnt;
  for (int i = lo; i < hi; ++i) {
    prefix[i] = run;
    run += need[i];
  }
  if (t == nt - 1) prefix[P] = run;
}
__global__ void k_need_counts(const int* prefix, const int* bounds, int G, int* counts) {
  const int r = threadIdx.x;
  if (r < G) counts[r] = prefix[bounds[r + 1]] - prefix[bounds[r]];
}
// this rank's needed genomes, in index order, into the send buffers
__global__ void k_pack(const int* need, const int* prefix, int lo, int hi, const double* pn, const double* pc,
                       double* send_n, double* send_c, int N, int C) {
  const int i = lo + blockIdx.x;
  if (i >= hi || !need[i]) return;
  const size_t gn = size_t(N) * kNodeCols, gc = size_t(C) * kConnCols;
  const size_t d = size_t(prefix[i] - prefix[lo]);
  const double2* a = reinterpret_cast<const double2*>(pn + size_t(i) * gn);
  const double2* b = reinterpret_cast<const double2*>(pc + size_t(i) * gc);
  double2* x = reinterpret_cast<double2*>(send_n + d * gn);
  double2* y = reinterpret_cast<double2*>(send_c + d * gc);
  for (size_t k = threadIdx.x; k < gn / 2; k += blockDim.x) x[k] = a[k];
  for (size_t k = threadIdx.x; k < gc / 2; k += blockDim.x) y[k] = b[k];
}
// parent indices -> positions in the gathered pool [G][M] genomes
__global__ void k_remap_parents(const int* fit_idx, const int* oth_idx, int P, const int* prefix, const int* bounds,
                                int G, int M, int* fitp, int* othp) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P) return;
  auto pos = [&](int g) {
    int r = 0;
    while (r + 1 < G && bounds[r + 1] <= g) ++r;
    return r * M + (prefix[g] - prefix[bounds[r]]);
  };
  fitp[c] = pos(fit_idx[c]);
  othp[c] = pos(oth_idx[c]);
}

// FNB_STEP_OVERLAP=0: the one-process step on one stream (A/B, debugging)
static bool step_overlap_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FNB_STEP_OVERLAP");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

struct Evolver {
  NeatCfg cfg;
  fnb_mutation_config mut;
  fnb_distance_config dist;
  DevShape sh;
  uint64_t seed = 0;
  int generation = 0;
  int P = 0, N = 0, C = 0;
  int host_species = 0;  // mirror of sd->count, refreshed at the end of a step
  cudaStream_t st = nullptr;
  long long* launches = nullptr;
  // device buffers
  double *pn[2] = {nullptr, nullptr}, *pc[2] = {nullptr, nullptr};
  int cur = 0;
  double* fitness = nullptr;
  double *rep_n = nullptr, *rep_c = nullptr;
  double* dmat = nullptr;
  int* species_of = nullptr;
  SpeciesDev* sd = nullptr;
  unsigned long long *kasc = nullptr, *kdesc = nullptr, *ktmp = nullptr;
  int *idx = nullptr, *idx_sorted = nullptr, *idx_tmp = nullptr, *skey = nullptr, *skey_tmp = nullptr;
  int *fit_idx = nullptr, *oth_idx = nullptr, *status = nullptr, *next_key = nullptr, *rank2 = nullptr;
  uint32_t *xkeys = nullptr, *mkeys = nullptr;
  uint8_t* active = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;

  size_t gn() const { return size_t(N) * kNodeCols; }
  size_t gc() const { return size_t(C) * kConnCols; }

  cudaError_t alloc() {
    cudaError_t e = cudaSuccess;
    auto A = [&](auto** p, size_t bytes) {
      if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
    };
    for (int b = 0; b < 2; ++b) {
      A(&pn[b], sizeof(double) * gn() * P);
      A(&pc[b], sizeof(double) * gc() * P);
    }
    A(&fitness, sizeof(double) * P);
    A(&rep_n, sizeof(double) * gn() * kMaxSpecies);
    A(&rep_c, sizeof(double) * gc() * kMaxSpecies);
    A(&dmat, sizeof(double) * size_t(P) * 2 * kMaxSpecies);  // [old reps | overflow vs all reps]
    A(&species_of, sizeof(int) * P);
    A(&sd, sizeof(SpeciesDev));
    A(&kasc, 8 * size_t(P));
    A(&kdesc, 8 * size_t(P));
    A(&ktmp, 8 * size_t(P));
    A(&idx, 4 * size_t(P));
    A(&idx_sorted, 4 * size_t(P));
    A(&idx_tmp, 4 * size_t(P));
    A(&skey, 4 * size_t(P));
    A(&skey_tmp, 4 * size_t(P));
    A(&fit_idx, 4 * size_t(P));
    A(&oth_idx, 4 * size_t(P));
    A(&status, 4 * size_t(P));
    A(&rank2, 4 * size_t(P));
    A(&next_key, 8);
    A(&xkeys, 16 * size_t(P));
    A(&mkeys, 16 * size_t(P));
    A(&active, size_t(P));
    if (e != cudaSuccess) return e;
    size_t b1 = 0, b2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b1, kasc, ktmp, idx, idx_tmp, P);
    cub::DeviceRadixSort::SortPairs(nullptr, b2, skey, skey_tmp, idx, idx_tmp, P, 0, 6);
    cub_bytes = std::max(b1, b2);
    A(&cub_tmp, cub_bytes);
    scratch_bytes = std::max(distance_scratch_bytes(kMaxSpecies, N, C), mutate_scratch_bytes(P, N, C));
    A(&scratch, scratch_bytes);
    if (e != cudaSuccess) return e;
    // representatives start as empty genomes (never read before founded)
    e = cudaMemsetAsync(rep_n, 0xff, sizeof(double) * gn() * kMaxSpecies, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(rep_c, 0xff, sizeof(double) * gc() * kMaxSpecies, st);
    SpeciesDev z{};
    if (e == cudaSuccess) e = cudaMemcpyAsync(sd, &z, sizeof(z), cudaMemcpyHostToDevice, st);
    const int nk[2] = {sh.I + sh.O + 1, 0};  // InnovationTable(first_key = I + O + 1)
    if (e == cudaSuccess) e = cudaMemcpyAsync(next_key, nk, sizeof(nk), cudaMemcpyHostToDevice, st);
    return e;
  }

  // one-process step (enqueue_step): two independent branches run on a side
  // stream -- the fitness sort next to speciation + stagnation, and the
  // mutation plans + K7 next to crossover -- joined by events (graph capture
  // turns them into parallel graph branches)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork[2] = {}, ev_join[2] = {};
  bool overlap = false;
  cudaError_t ensure_side() {
    if (side) return cudaSuccess;
    cudaError_t e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&ev_fork[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_join[i], cudaEventDisableTiming);
    }
    return e;
  }

  void release() {
    release_graphs();
    shard_release();
    for (int i = 0; i < 2; ++i) {
      if (ev_fork[i]) cudaEventDestroy(ev_fork[i]);
      if (ev_join[i]) cudaEventDestroy(ev_join[i]);
    }
    if (side) cudaStreamDestroy(side);
    void* ps[] = {pn[0], pn[1], pc[0], pc[1], fitness, rep_n, rep_c, dmat, species_of, sd,
                  kasc, kdesc, ktmp, idx, idx_sorted, idx_tmp, skey, skey_tmp, fit_idx, oth_idx, status, next_key, rank2,
                  xkeys, mkeys, active, cub_tmp, scratch};
    for (void* p : ps)
      if (p) cudaFree(p);
  }

  cudaError_t init_population() {
    const Key4 root = key_from_seed(seed);
    k_init_population<<<(P + 3) / 4, 128, 0, st>>>(pn[cur], pc[cur], P, N, C, sh.I, sh.O, key_split(root, 0),
                                                   mut.bias.init_mean, mut.bias.init_std, mut.response.init_mean,
                                                   mut.response.init_std, mut.weight.init_mean, mut.weight.init_std,
                                                   sh.default_agg, sh.default_act, cfg.output_activation);
    ++*launches;
    return cudaGetLastError();
  }

  int coop_blocks = 0;  // co-resident CTAs of k_found_rounds (cooperative launch bound)

  cudaError_t launch_found_rounds(int S_old, const double* n, const double* c) {
    int Hn = table_capacity(N), Hc = table_capacity(C);
    const int block = 128;
    const size_t smem = size_t(Hn) * 12 + size_t(Hc) * 20 + 16 + (block / 32) * 8 + (block / 32) * 33 * 8;
    cudaError_t e = cudaFuncSetAttribute(k_found_rounds, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    if (coop_blocks == 0) {
      int dev = 0, sms = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_found_rounds, block, smem);
      if (e != cudaSuccess) return e;
      coop_blocks = std::max(1, per_sm * sms);
    }
    int grid = std::max(1, std::min(coop_blocks, (P + block / 32 - 1) / (block / 32)));
    int ms = cfg.max_species;
    double th = cfg.threshold, cd = dist.compatibility_disjoint, ch = dist.compatibility_homologous;
    int p = P, nn = N, cc = C;
    void* args[] = {&sd, &S_old, &ms, &species_of, &n, &c, &rep_n, &rep_c, &p, &nn, &cc, &th, &cd, &ch, &Hn, &Hc};
    ++*launches;
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_found_rounds), dim3(grid), dim3(block), args, smem,
                                       st);
  }

  // One generation step = enqueue_step() (all kernels, no host sync) and a
  // 12-byte status read.  The kernel sequence depends only on (S_old, cur),
  // so it is captured once per pair as a CUDA graph and replayed; the
  // generation number the keys need lives in SpeciesDev.  FNB_STEP_GRAPH=0
  // (or a failed capture) runs the same sequence eagerly.
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    long long n_launches = 0;
  };
  StepGraph graphs[kMaxSpecies + 1][2];
  bool use_graphs = true;

  cudaError_t step(int* host_error) {
    cudaError_t e = cudaSuccess;
    if (use_graphs) {
      StepGraph& g = graphs[host_species][cur];
      if (!g.exec) {
        const long long before = *launches;
        cudaGraph_t graph = nullptr;
        e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
          const cudaError_t ee = enqueue_step();
          e = cudaStreamEndCapture(st, &graph);
          if (ee != cudaSuccess) e = ee;
        }
        if (e == cudaSuccess) e = cudaGraphInstantiate(&g.exec, graph, 0);
        g.n_launches = *launches - before;
        *launches = before;
        if (e == cudaSuccess) {  // exact: the kernel nodes the capture recorded
          size_t n = 0;
          if (cudaGraphGetNodes(graph, nullptr, &n) == cudaSuccess) {
            std::vector<cudaGraphNode_t> nodes(n);
            long long k = 0;
            if (n && cudaGraphGetNodes(graph, nodes.data(), &n) == cudaSuccess) {
              for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType t;
                if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
              }
              g.n_launches = k;
            }
          }
        }
        if (graph) cudaGraphDestroy(graph);
        if (e != cudaSuccess) {  // e.g. a capture-unsupported launch: stay eager
          g.exec = nullptr;
          use_graphs = false;
          cudaGetLastError();
        }
      }
      if (use_graphs) {
        e = cudaGraphLaunch(g.exec, st);
        if (e != cudaSuccess) return e;
        *launches += g.n_launches;
      }
    }
    if (!use_graphs) {
      e = enqueue_step();
      if (e != cudaSuccess) return e;
    }
    return read_status_and_swap(host_error);
  }

  // 12-byte status read after a step; the next buffer becomes current
  cudaError_t read_status_and_swap(int* host_error) {
    cudaError_t e;
    int stat[3] = {0, 0, INT_MAX};  // error, count, first_bad
    e = cudaMemcpyAsync(&stat[0], &sd->error, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&stat[1], &sd->count, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&stat[2], &sd->first_bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    *host_error = stat[0] ? -2 : (stat[2] == INT_MAX ? -1 : stat[2]);
    host_species = stat[1];
    cur ^= 1;
    ++generation;
    return cudaSuccess;
  }

  void release_graphs() {
    for (auto& row : graphs)
      for (auto& g : row)
        if (g.exec) {
          cudaGraphExecDestroy(g.exec);
          g.exec = nullptr;
        }
  }

  // speciate -> update_stagnation -> compute_spawn_counts -> parent
  // selection -> mutation plans + innovation keys (all slots)
  cudaError_t enqueue_front() {
    const int T = 256, B = (P + T - 1) / T;
    const double th = cfg.threshold;
    const double* n = pn[cur];
    const double* c = pc[cur];
    cudaError_t e;
    const int S_old = host_species;
    const bool ov = overlap;
    // the fitness order (ranks by a stable ascending sort, members by fitness
    // desc / index asc) needs only the fitness: on the side stream, next to
    // speciation and stagnation
    auto fitness_sort = [&](cudaStream_t s) -> cudaError_t {
      k_fit_keys<<<B, T, 0, s>>>(fitness, P, kasc, kdesc, idx);
      cudaError_t r = P <= kCountRankMax
                          ? launch_count_sort<unsigned long long>(kasc, nullptr, P, skey_tmp, ktmp, idx_sorted, s)
                          : cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, kasc, ktmp, idx, idx_sorted, P, 0, 64, s);
      if (r != cudaSuccess) return r;
      k_desc_from_asc<<<B, T, 0, s>>>(ktmp, idx_sorted, P, idx_tmp, rank2);
      return cudaGetLastError();
    };
    if (ov) {
      e = cudaEventRecord(ev_fork[0], st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ev_fork[0], 0);
      if (e == cudaSuccess) e = fitness_sort(side);
      if (e == cudaSuccess) e = cudaEventRecord(ev_join[0], side);
      if (e != cudaSuccess) return e;
    }
    // ---- speciate
    k_spec_begin<<<1, 1, 0, st>>>(sd);
    if (S_old > 0) {
      e = launch_distance_masked(n, c, P, rep_n, rep_c, S_old, N, C, dist.compatibility_disjoint,
                                 dist.compatibility_homologous, dmat, scratch, scratch_bytes, nullptr, nullptr, st);
      if (e != cudaSuccess) return e;
    }
    k_assign_first<<<B, T, 0, st>>>(dmat, 0, P, S_old, th, species_of);
    *launches += 2 + (S_old > 0 ? kDistanceLaunches : 0);
    if (S_old < cfg.max_species) {
      e = launch_found_rounds(S_old, n, c);
      if (e != cudaSuccess) return e;
    }
    e = launch_distance_masked(n, c, P, rep_n, rep_c, cfg.max_species, N, C, dist.compatibility_disjoint,
                               dist.compatibility_homologous, dmat + size_t(P) * S_old, scratch, scratch_bytes,
                               species_of, nullptr, st);
    if (e != cudaSuccess) return e;
    k_nearest<<<B, T, 0, st>>>(dmat + size_t(P) * S_old, 0, P, cfg.max_species, sd, species_of);
    if (S_old > 0) {
      k_rep_min<<<B, T, 0, st>>>(dmat, 0, P, S_old, species_of, sd, 0);
      k_rep_min<<<B, T, 0, st>>>(dmat, 0, P, S_old, species_of, sd, 1);
      k_rep_copy<<<S_old, 256, 0, st>>>(sd, n, c, rep_n, rep_c, N, C);
    }
    k_sizes<<<B, T, 0, st>>>(species_of, 0, P, sd);
    k_mark_nonempty<<<1, 1, 0, st>>>(sd);
    k_apply_compaction<<<1, 256, 0, st>>>(sd, rep_n, rep_c, N, C);
    k_remap<<<B, T, 0, st>>>(species_of, 0, P, sd);
    // ---- update_stagnation
    k_stag_begin<<<1, 1, 0, st>>>(sd);
    k_species_max<<<B, T, 0, st>>>(fitness, species_of, 0, P, sd);
    k_stagnation<<<1, 1, 0, st>>>(sd, cfg.species_elitism, cfg.max_stagnation);
    k_apply_compaction<<<1, 256, 0, st>>>(sd, rep_n, rep_c, N, C);
    k_remap_or_drop<<<B, T, 0, st>>>(species_of, 0, P, sd);
    // ---- compute_spawn_counts: ranks by a stable ascending sort; members by
    //      (fitness desc, index asc) for reproduce, and the mid-ranks
    if (!ov) {
      e = fitness_sort(st);
      if (e != cudaSuccess) return e;
    }
    k_spawn_begin<<<1, 1, 0, st>>>(sd);
    if (ov) {
      e = cudaStreamWaitEvent(st, ev_join[0], 0);
      if (e != cudaSuccess) return e;
    }
    k_rank_sums<<<B, T, 0, st>>>(rank2, idx_sorted, P, species_of, 0, P, sd);
    k_spawn<<<1, 1, 0, st>>>(sd, P, cfg.spawn_rate, cfg.genome_elitism);
    // ---- reproduce: members by species
    k_species_keys<<<B, T, 0, st>>>(idx_tmp, P, species_of, skey);
    e = P <= kCountRankMax
            ? launch_count_sort<int>(skey, idx_tmp, P, skey_tmp, nullptr, idx_sorted, st)
            : cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, skey, skey_tmp, idx_tmp, idx_sorted, P, 0, 6, st);
    if (e != cudaSuccess) return e;
    const Key4 root1 = key_split(key_from_seed(seed), 1);
    k_reproduce_plan<<<B, T, 0, st>>>(sd, idx_sorted, fitness, P, root1, cfg.genome_elitism, cfg.survival, fit_idx,
                                      oth_idx, xkeys, mkeys, active);
    *launches += 22 + kDistanceLaunches;
    // mutate phase 1 over all slots (replicated on every rank of a sharded
    // run): node-split plans read from the fit parents, K7 innovation keys;
    // in the one-process step on the side stream, next to crossover
    if (ov) {
      e = cudaEventRecord(ev_fork[1], st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ev_fork[1], 0);
      if (e == cudaSuccess)
        e = launch_mutate_plan(n, c, fit_idx, mkeys, P, active, &mut, sh, next_key, scratch, scratch_bytes, nullptr,
                               side, launches);
      if (e == cudaSuccess) e = cudaEventRecord(ev_join[1], side);
      return e;
    }
    e = launch_mutate_plan(n, c, fit_idx, mkeys, P, active, &mut, sh, next_key, scratch, scratch_bytes, nullptr, st,
                           launches);
    return e;
  }

  // Children [lo, hi) into the next buffer: crossover (K5), then structural
  // and attribute mutation (K6) with the keys planned by enqueue_front.
  cudaError_t enqueue_back(int lo, int hi) {
    if (hi <= lo) return cudaSuccess;
    const double* n = pn[cur];
    const double* c = pc[cur];
    cudaError_t e = launch_crossover(n, c, fit_idx + lo, oth_idx + lo, xkeys + 4 * size_t(lo), hi - lo, N, C,
                                     pn[cur ^ 1] + size_t(lo) * gn(), pc[cur ^ 1] + size_t(lo) * gc(), st);
    if (e != cudaSuccess) return e;
    ++*launches;
    if (overlap) {  // the mutation plans (side stream) before the structural pass
      e = cudaStreamWaitEvent(st, ev_join[1], 0);
      if (e != cudaSuccess) return e;
    }
    int* newk = mutate_new_keys();
    return launch_mutate_apply(pn[cur ^ 1], pc[cur ^ 1], mkeys, P, lo, hi, active, &mut, sh, status, scratch,
                               scratch_bytes, newk, st, launches);
  }

  // the K7 key array inside the mutate scratch (layout of mutate.cu mut_scratch)
  int* mutate_new_keys() const {
    const size_t H = size_t(table_capacity(P));
    return reinterpret_cast<int*>(static_cast<uint8_t*>(scratch) + size_t(P) * 8 + H * 8 + size_t(P) * 8);
  }

  // lowest failing slot among the slots this process produced
  cudaError_t enqueue_first_bad(int lo, int hi) {
    const int T = 256;
    if (hi > lo) {
      k_first_bad<<<(hi - lo + T - 1) / T, T, 0, st>>>(status + lo, hi - lo, sd, lo);
      ++*launches;
    }
    return cudaGetLastError();
  }
  // once per generation: the device generation counter the key tree reads
  cudaError_t enqueue_advance() {
    k_gen_advance<<<1, 1, 0, st>>>(sd);
    ++*launches;
    return cudaGetLastError();
  }

  // speciate -> update_stagnation -> compute_spawn_counts -> reproduce
  cudaError_t enqueue_step() {
    cudaError_t e = step_overlap_enabled() ? ensure_side() : cudaSuccess;
    overlap = e == cudaSuccess && step_overlap_enabled();
    if (e == cudaSuccess) e = enqueue_front();
    if (e == cudaSuccess) e = enqueue_back(0, P);
    overlap = false;
    if (e == cudaSuccess) e = enqueue_first_bad(0, P);
    if (e == cudaSuccess) e = enqueue_advance();
    return e;
  }

  // Sharded reproduction (distributed.py): every rank runs the front on the
  // replicated population, produces children [lo, hi) (any number of
  // back calls over disjoint ranges) and the caller all-gathers the next
  // buffer before commit().
  cudaError_t front_eager() { return enqueue_front(); }
  cudaError_t back_eager(int lo, int hi) {
    cudaError_t e = enqueue_back(lo, hi);
    if (e == cudaSuccess) e = enqueue_first_bad(lo, hi);
    return e;
  }
  cudaError_t commit(int* host_error) {
    cudaError_t e = enqueue_advance();
    return e == cudaSuccess ? read_status_and_swap(host_error) : e;
  }

  // ---- the sharded step: buffers and phases (fnb_evolver_shard_phase) ----------------
  int sh_world = 0;
  std::vector<int> sh_bounds;                   // host copy, world + 1
  int* d_bounds = nullptr;                      // device copy
  int *need = nullptr, *prefix = nullptr, *counts = nullptr, *fitp = nullptr, *othp = nullptr, *min_u = nullptr;
  double* dfound = nullptr;
  unsigned long long* stage = nullptr;
  double *send_n = nullptr, *send_c = nullptr, *pool_n = nullptr, *pool_c = nullptr;
  size_t send_cap = 0, pool_cap = 0;            // genomes

  cudaError_t shard_init(int world, const int* bounds) {
    cudaError_t e = cudaSuccess;
    auto A = [&](auto** p, size_t bytes) {
      if (e == cudaSuccess && !*p) e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
    };
    A(&need, 4 * size_t(P));
    A(&prefix, 4 * (size_t(P) + 1));
    A(&fitp, 4 * size_t(P));
    A(&othp, 4 * size_t(P));
    A(&min_u, 16);
    A(&dfound, 8 * size_t(P));
    A(&stage, 8 * (gn() + gc()) * kMaxSpecies);
    if (e == cudaSuccess && world != sh_world) {
      if (d_bounds) cudaFree(d_bounds);
      if (counts) cudaFree(counts);
      d_bounds = nullptr;
      counts = nullptr;
      A(&d_bounds, 4 * (size_t(world) + 1));
      A(&counts, 4 * size_t(world));
    }
    if (e != cudaSuccess) return e;
    sh_world = world;
    sh_bounds.assign(bounds, bounds + world + 1);
    return cudaMemcpyAsync(d_bounds, bounds, 4 * (size_t(world) + 1), cudaMemcpyHostToDevice, st);
  }
  void shard_release() {
    void* ps[] = {need, prefix, fitp, othp, min_u, dfound, stage, d_bounds, counts, send_n, send_c, pool_n, pool_c};
    for (void* p : ps)
      if (p) cudaFree(p);
  }
  cudaError_t ensure_genomes(double** pn_, double** pc_, size_t* cap, size_t n) {
    if (n <= *cap) return cudaSuccess;
    if (*pn_) cudaFree(*pn_);
    if (*pc_) cudaFree(*pc_);
    *pn_ = *pc_ = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(pn_), 8 * gn() * n);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(pc_), 8 * gc() * n);
    if (e == cudaSuccess) *cap = n;
    return e;
  }

  // phase 0: speciate begins -- first match against the old representatives
  cudaError_t shard_begin(int lo, int hi) {
    const int T = 256, B = (hi - lo + T - 1) / T;
    const int S_old = host_species;
    const double* n = pn[cur];
    const double* c = pc[cur];
    k_spec_begin<<<1, 1, 0, st>>>(sd);
    ++*launches;
    if (hi <= lo) return cudaGetLastError();
    if (S_old > 0) {
      cudaError_t e = launch_distance_masked(n + size_t(lo) * gn(), c + size_t(lo) * gc(), hi - lo, rep_n, rep_c, S_old,
                                             N, C, dist.compatibility_disjoint, dist.compatibility_homologous,
                                             dmat + size_t(lo) * S_old, scratch, scratch_bytes, nullptr, nullptr, st);
      if (e != cudaSuccess) return e;
      *launches += kDistanceLaunches;
    }
    k_assign_first<<<B, T, 0, st>>>(dmat, lo, hi, S_old, cfg.threshold, species_of);
    ++*launches;
    return cudaGetLastError();
  }
  // phase 1: lowest unassigned genome of this shard -> min_u[0] (INT_MAX none)
  cudaError_t shard_min_unassigned(int lo, int hi) {
    k_set_int<<<1, 1, 0, st>>>(min_u, INT_MAX);
    if (hi > lo) k_min_unassigned<<<(hi - lo + 255) / 256, 256, 0, st>>>(species_of, lo, hi, min_u);
    *launches += 1 + (hi > lo);
    return cudaGetLastError();
  }
  // phase 2 (the founder's owner): representative slot j <- genome f
  cudaError_t shard_found(int f, int j) {
    k_found_copy<<<1, 256, 0, st>>>(pn[cur], pc[cur], f, j, rep_n, rep_c, species_of, N, C);
    ++*launches;
    return cudaGetLastError();
  }
  // phase 3 (every rank, after the broadcast of slot j): commit species j and
  // join the shard's unassigned genomes within the threshold of its founder
  cudaError_t shard_join(int lo, int hi, int j) {
    k_found_commit<<<1, 1, 0, st>>>(sd, j);
    ++*launches;
    if (hi > lo) {
      cudaError_t e = launch_distance_masked(pn[cur] + size_t(lo) * gn(), pc[cur] + size_t(lo) * gc(), hi - lo,
                                             rep_n + size_t(j) * gn(), rep_c + size_t(j) * gc(), 1, N, C,
                                             dist.compatibility_disjoint, dist.compatibility_homologous, dfound + lo,
                                             scratch, scratch_bytes, species_of + lo, nullptr, st);
      if (e != cudaSuccess) return e;
      k_join<<<(hi - lo + 255) / 256, 256, 0, st>>>(dfound, lo, hi, cfg.threshold, j, species_of);
      *launches += kDistanceLaunches + 1;
    }
    return cudaGetLastError();
  }
  // phase 4: nearest-representative overflow, then pass 0 of the new
  // representative search (min distance bits per old species -> sd->dmin)
  cudaError_t shard_assign_rest(int lo, int hi) {
    const int T = 256, B = (hi - lo + T - 1) / T;
    const int S_old = host_species;
    if (hi <= lo) return cudaSuccess;
    cudaError_t e = launch_distance_masked(pn[cur] + size_t(lo) * gn(), pc[cur] + size_t(lo) * gc(), hi - lo, rep_n,
                                           rep_c, cfg.max_species, N, C, dist.compatibility_disjoint,
                                           dist.compatibility_homologous,
                                           dmat + size_t(P) * S_old + size_t(lo) * cfg.max_species, scratch,
                                           scratch_bytes, species_of + lo, nullptr, st);
    if (e != cudaSuccess) return e;
    k_nearest<<<B, T, 0, st>>>(dmat + size_t(P) * S_old, lo, hi, cfg.max_species, sd, species_of);
    *launches += kDistanceLaunches + 1;
    if (S_old > 0) {
      k_rep_min<<<B, T, 0, st>>>(dmat, lo, hi, S_old, species_of, sd, 0);
      ++*launches;
    }
    return cudaGetLastError();
  }
  // phase 5: pass 1 (lowest index at the minimum -> sd->argmin)
  cudaError_t shard_rep_argmin(int lo, int hi) {
    const int S_old = host_species;
    if (S_old > 0 && hi > lo) {
      k_rep_min<<<(hi - lo + 255) / 256, 256, 0, st>>>(dmat, lo, hi, S_old, species_of, sd, 1);
      ++*launches;
    }
    return cudaGetLastError();
  }
  // phase 6: stage the new representatives this shard owns (zeros elsewhere)
  cudaError_t shard_rep_stage(int lo, int hi) {
    const int S_old = host_species;
    if (S_old > 0) {
      k_rep_stage<<<S_old, 256, 0, st>>>(sd, pn[cur], pc[cur], lo, hi, stage, N, C);
      ++*launches;
    }
    return cudaGetLastError();
  }
  // phase 7: commit the summed stage; species sizes of the shard (-> sd->size)
  cudaError_t shard_rep_commit(int lo, int hi) {
    const int S_old = host_species;
    if (S_old > 0) {
      k_rep_commit<<<S_old, 256, 0, st>>>(sd, stage, rep_n, rep_c, N, C);
      ++*launches;
    }
    if (hi > lo) {
      k_sizes<<<(hi - lo + 255) / 256, 256, 0, st>>>(species_of, lo, hi, sd);
      ++*launches;
    }
    return cudaGetLastError();
  }
  // phase 8: drop empty species; species max fitness of the shard (-> sd->mxbits)
  cudaError_t shard_compact(int lo, int hi) {
    const int T = 256, B = (hi - lo + T - 1) / T;
    k_mark_nonempty<<<1, 1, 0, st>>>(sd);
    k_apply_compaction<<<1, 256, 0, st>>>(sd, rep_n, rep_c, N, C);
    k_stag_begin<<<1, 1, 0, st>>>(sd);
    *launches += 3;
    if (hi > lo) {
      k_remap<<<B, T, 0, st>>>(species_of, lo, hi, sd);
      k_species_max<<<B, T, 0, st>>>(fitness, species_of, lo, hi, sd);
      *launches += 2;
    }
    return cudaGetLastError();
  }
  // phase 9: stagnation (replicated); fitness ranks over the whole gathered
  // vector, mid-rank sums of the shard's genomes (-> sd->rsum, sd->cnt)
  cudaError_t shard_stagnation(int lo, int hi) {
    const int T = 256, B = (P + T - 1) / T;
    k_stagnation<<<1, 1, 0, st>>>(sd, cfg.species_elitism, cfg.max_stagnation);
    k_apply_compaction<<<1, 256, 0, st>>>(sd, rep_n, rep_c, N, C);
    if (hi > lo) k_remap_or_drop<<<(hi - lo + T - 1) / T, T, 0, st>>>(species_of, lo, hi, sd);
    k_fit_keys<<<B, T, 0, st>>>(fitness, P, kasc, kdesc, idx);
    cudaError_t e = P <= kCountRankMax
                        ? launch_count_sort<unsigned long long>(kasc, nullptr, P, skey_tmp, ktmp, idx_sorted, st)
                        : cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, kasc, ktmp, idx, idx_sorted, P, 0, 64, st);
    if (e != cudaSuccess) return e;
    k_spawn_begin<<<1, 1, 0, st>>>(sd);
    k_desc_from_asc<<<B, T, 0, st>>>(ktmp, idx_sorted, P, idx_tmp, rank2);
    k_rank_sums<<<B, T, 0, st>>>(rank2, idx_sorted, P, species_of, lo, hi, sd);
    *launches += 9 + (hi > lo);
    return cudaGetLastError();
  }
  // phase 10 (after the all-gather of species_of): spawn, members, parent
  // selection for every slot, the parents' pool positions; counts[r] = the
  // parents rank r holds
  cudaError_t shard_select() {
    const int T = 256, B = (P + T - 1) / T;
    k_spawn<<<1, 1, 0, st>>>(sd, P, cfg.spawn_rate, cfg.genome_elitism);
    k_species_keys<<<B, T, 0, st>>>(idx_tmp, P, species_of, skey);
    cudaError_t e = P <= kCountRankMax
                        ? launch_count_sort<int>(skey, idx_tmp, P, skey_tmp, nullptr, idx_sorted, st)
                        : cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, skey, skey_tmp, idx_tmp, idx_sorted, P,
                                                          0, 6, st);
    if (e != cudaSuccess) return e;
    const Key4 root1 = key_split(key_from_seed(seed), 1);
    k_reproduce_plan<<<B, T, 0, st>>>(sd, idx_sorted, fitness, P, root1, cfg.genome_elitism, cfg.survival, fit_idx,
                                      oth_idx, xkeys, mkeys, active);
    e = cudaMemsetAsync(need, 0, 4 * size_t(P), st);
    if (e != cudaSuccess) return e;
    k_need<<<B, T, 0, st>>>(fit_idx, oth_idx, P, need);
    k_scan_need<<<1, 1024, 0, st>>>(need, P, prefix);
    k_need_counts<<<1, 32 * ((sh_world + 31) / 32), 0, st>>>(prefix, d_bounds, sh_world, counts);
    *launches += 8;
    return cudaGetLastError();
  }
  // phase 11: the shard's parents into the send buffers (M genomes each)
  cudaError_t shard_pack(int lo, int hi, int M) {
    cudaError_t e = ensure_genomes(&send_n, &send_c, &send_cap, size_t(std::max(M, 1)));
    if (e == cudaSuccess) e = ensure_genomes(&pool_n, &pool_c, &pool_cap, size_t(std::max(M, 1)) * sh_world);
    if (e != cudaSuccess) return e;
    if (hi > lo) {
      k_pack<<<hi - lo, 128, 0, st>>>(need, prefix, lo, hi, pn[cur], pc[cur], send_n, send_c, N, C);
      ++*launches;
    }
    return cudaGetLastError();
  }
  // phase 12 (after the all-gather of the send buffers into the pool):
  // node-split plans and innovation keys for ALL slots from the pool
  // (replicated), then crossover + mutation of the shard's children
  cudaError_t shard_back(int lo, int hi, int M) {
    const int T = 256, B = (P + T - 1) / T;
    k_remap_parents<<<B, T, 0, st>>>(fit_idx, oth_idx, P, prefix, d_bounds, sh_world, M, fitp, othp);
    ++*launches;
    cudaError_t e = launch_mutate_plan(pool_n, pool_c, fitp, mkeys, P, active, &mut, sh, next_key, scratch,
                                       scratch_bytes, nullptr, st, launches);
    if (e != cudaSuccess || hi <= lo) return e;
    e = launch_crossover(pool_n, pool_c, fitp + lo, othp + lo, xkeys + 4 * size_t(lo), hi - lo, N, C,
                         pn[cur ^ 1] + size_t(lo) * gn(), pc[cur ^ 1] + size_t(lo) * gc(), st);
    if (e != cudaSuccess) return e;
    ++*launches;
    e = launch_mutate_apply(pn[cur ^ 1], pc[cur ^ 1], mkeys, P, lo, hi, active, &mut, sh, status, scratch,
                            scratch_bytes, mutate_new_keys(), st, launches);
    if (e != cudaSuccess) return e;
    return enqueue_first_bad(lo, hi);
  }
};

}  // namespace fnb

// =================================================================================
// C ABI: fnb_evolver_* (include/flatneat_b200.h)
// =================================================================================
#include "ctx_internal.cuh"

struct fnb_evolve_run;
static void release_evolve_run(fnb_evolve_run* r);

struct fnb_evolver {
  fnb_ctx* ctx = nullptr;
  fnb::Evolver ev;
  DevBuf nets, X, Y;
  // evaluation status (written on the evolver stream, read by eval_check):
  // [0] lowest genome whose transform failed (INT_MAX none), [1] non-finite X
  DevBuf eflags;
  int eval_lo = 0, eval_n = 0;
  int run_mode = -1;  // fnb_evolve: 2 conditional generation graphs, 1 evaluate graph + step graph, 0 eager
  struct fnb_evolve_run* run = nullptr;  // generation graphs, kept across fnb_evolve calls
};

namespace fnb {
int launch_forward(const void* nets, NetLayout L, int P, const float* X, const float* Y, int B, int fit_kind,
                   double offset, double* fitness, double* out, double* partial_buf, size_t partial_cap,
                   int uniform_agg, int uniform_act, cudaStream_t st, long long* launches);
size_t forward_partial_needed(NetLayout L, int P, int B);
cudaError_t launch_transform(const double* n, const double* c, int P, uint8_t* nets, const NetLayout& L,
                             const DevShape& sh, cudaStream_t st);
}  // namespace fnb

namespace fnb {
cudaError_t launch_first_error(const uint8_t* nets, size_t stride, int P, int* out, cudaStream_t st);

__global__ void k_eval_flags_init(int* f) {
  f[0] = INT_MAX;
  f[1] = 0;
}
// network.hpp:245-246: every input must be finite
__global__ void k_nonfinite_f32(const float* __restrict__ x, size_t n, int* bad) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    if (!isfinite(x[i])) atomicOr(bad, 1);
}

cudaError_t launch_validate(const double* nodes, const double* conns, int P, const DevShape& sh, int32_t* codes,
                            int32_t* details, cudaStream_t st);
std::string validate_message(int code, int detail);
}  // namespace fnb

#define EV_CK(expr)                                                         \
  do {                                                                      \
    cudaError_t e_ = (expr);                                                \
    if (e_ != cudaSuccess) return fnb_cuda_error(ev->ctx, e_, #expr);       \
  } while (0)

extern "C" {

int fnb_evolver_create(fnb_ctx* ctx, const fnb_neat_config* cfg, uint64_t seed, fnb_evolver** out) {
  if (!ctx || !cfg || !out) return 1 + FNB_E_CONFIG_ERROR;
  *out = nullptr;
  const fnb::DevShape& sh = ctx->sh;
  if (cfg->pop_size < 2 || cfg->max_species < 1 || cfg->max_species > fnb::kMaxSpecies ||
      cfg->survival_threshold <= 0.0 || cfg->survival_threshold > 1.0 ||
      cfg->max_species * cfg->genome_elitism > cfg->pop_size)
    return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "invalid NeatConfig", -1);
  if (sh.I + sh.O + 1 > sh.N || sh.I + sh.O > sh.C)
    return fnb_set_error(ctx, FNB_E_LIMITS_TOO_SMALL, "limits cannot hold the minimal genome", -1);
  for (int i = 0; i < sh.I; ++i)
    if (sh.input_keys[i] != i) return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "input keys must be 0..I-1", -1);
  for (int o = 0; o < sh.O; ++o)
    if (sh.output_keys[o] != sh.I + o)
      return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "output keys must be I..I+O-1", -1);
  if (cfg->output_activation < 0 || cfg->output_activation >= sh.n_act)
    return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "output activation id out of range", -1);
  auto* e = new fnb_evolver();
  e->ctx = ctx;
  fnb::Evolver& v = e->ev;
  v.cfg = fnb::NeatCfg{cfg->pop_size, cfg->max_species, cfg->compatibility_threshold, cfg->species_elitism,
                       cfg->max_stagnation, cfg->genome_elitism, cfg->survival_threshold,
                       cfg->spawn_number_change_rate, cfg->output_activation};
  v.mut = cfg->mutation;
  v.dist = cfg->distance;
  v.sh = sh;
  v.seed = seed;
  v.P = cfg->pop_size;
  v.N = sh.N;
  v.C = sh.C;
  v.st = ctx->stream;
  if (const char* g = std::getenv("FNB_STEP_GRAPH")) v.use_graphs = std::string(g) != "0";
  v.launches = &ctx->launches;
  cudaSetDevice(ctx->device);
  cudaError_t err = v.alloc();
  if (err == cudaSuccess) err = cudaStreamSynchronize(v.st);
  if (err != cudaSuccess) {
    v.release();
    delete e;
    return fnb_cuda_error(ctx, err, "evolver allocation");
  }
  *out = e;
  return 0;
}

void fnb_evolver_destroy(fnb_evolver* ev) {
  if (!ev) return;
  cudaSetDevice(ev->ctx->device);
  ev->ev.release();
  ev->nets.release();
  ev->X.release();
  ev->Y.release();
  ev->eflags.release();
  release_evolve_run(ev->run);
  delete ev;
  cudaGetLastError();  // leave no error behind for the context's next call
}

int fnb_evolver_init_population(fnb_evolver* ev) {
  cudaSetDevice(ev->ctx->device);
  EV_CK(ev->ev.init_population());
  EV_CK(cudaStreamSynchronize(ev->ev.st));
  return 0;
}

int fnb_evolver_set_population(fnb_evolver* ev, const double* nodes, const double* conns) {
  fnb::Evolver& v = ev->ev;
  cudaSetDevice(ev->ctx->device);
  // cudaMemcpyDefault: host or device (UVA) source
  EV_CK(cudaMemcpyAsync(v.pn[v.cur], nodes, sizeof(double) * v.gn() * v.P, cudaMemcpyDefault, v.st));
  EV_CK(cudaMemcpyAsync(v.pc[v.cur], conns, sizeof(double) * v.gc() * v.P, cudaMemcpyDefault, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  return 0;
}

int fnb_evolver_get_population(fnb_evolver* ev, double* nodes, double* conns) {
  fnb::Evolver& v = ev->ev;
  cudaSetDevice(ev->ctx->device);
  if (nodes) EV_CK(cudaMemcpyAsync(nodes, v.pn[v.cur], sizeof(double) * v.gn() * v.P, cudaMemcpyDefault, v.st));
  if (conns) EV_CK(cudaMemcpyAsync(conns, v.pc[v.cur], sizeof(double) * v.gc() * v.P, cudaMemcpyDefault, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  return 0;
}

int fnb_evolver_set_fitness(fnb_evolver* ev, const double* fitness) {
  fnb::Evolver& v = ev->ev;
  cudaSetDevice(ev->ctx->device);
  EV_CK(cudaMemcpyAsync(v.fitness, fitness, sizeof(double) * v.P, cudaMemcpyHostToDevice, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  return 0;
}

int fnb_evolver_get_fitness(fnb_evolver* ev, double* fitness) {
  fnb::Evolver& v = ev->ev;
  cudaSetDevice(ev->ctx->device);
  EV_CK(cudaMemcpyAsync(fitness, v.fitness, sizeof(double) * v.P, cudaMemcpyDeviceToHost, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  return 0;
}

// transform + forward + fused fitness of genomes [lo, lo+n) of the current
// population into d_fit, plus the evaluation status words (eflags) that
// fnb_evolver_eval_check reads: everything is enqueued on the evolver stream
// with no host synchronisation (capture-safe).
static int evolver_eval_enqueue(fnb_evolver* ev, int lo, int n, const float* d_X, const float* d_Y, int batch,
                                int fitness_kind, double fitness_offset, double* d_fit) {
  fnb::Evolver& v = ev->ev;
  fnb_ctx* ctx = ev->ctx;
  cudaSetDevice(ctx->device);
  if (batch <= 0) return fnb_set_error(ctx, FNB_E_EMPTY_DATASET, "batch is empty", -1);
  EV_CK(ev->nets.ensure(ctx->L.bytes * size_t(std::max(n, 1))));
  EV_CK(ev->eflags.ensure(4 * sizeof(int)));
  int* fl = static_cast<int*>(ev->eflags.p);
  ev->eval_lo = lo;
  ev->eval_n = n;
  fnb::k_eval_flags_init<<<1, 1, 0, v.st>>>(fl);
  ++ctx->launches;
  const size_t nx = size_t(batch) * ctx->sh.I;
  if (nx > 0) {
    fnb::k_nonfinite_f32<<<int(std::min<size_t>((nx + 255) / 256, 148)), 256, 0, v.st>>>(d_X, nx, fl + 1);
    ++ctx->launches;
  }
  if (n == 0) return 0;
  EV_CK(fnb::launch_transform(v.pn[v.cur] + size_t(lo) * v.gn(), v.pc[v.cur] + size_t(lo) * v.gc(), n,
                              static_cast<uint8_t*>(ev->nets.p), ctx->L, ctx->sh, v.st));
  ctx->launches++;
  EV_CK(ctx->partial.ensure(fnb::forward_partial_needed(ctx->L, n, batch)));
  // genomes that failed K1 are skipped by K2 (their fitness is not written)
  if (fnb::launch_forward(ev->nets.p, ctx->L, n, d_X, d_Y, batch, fitness_kind, fitness_offset, d_fit, nullptr,
                          static_cast<double*>(ctx->partial.p), ctx->partial.cap,
                          ctx->sh.n_agg == 1 ? int(ctx->sh.agg[0]) : -1, ctx->sh.n_act == 1 ? int(ctx->sh.act[0]) : -1,
                          v.st, &ctx->launches))
    return fnb_cuda_error(ctx, cudaGetLastError(), "forward launch");
  EV_CK(fnb::launch_first_error(static_cast<const uint8_t*>(ev->nets.p), ctx->L.bytes, n, fl, v.st));
  ctx->launches++;
  return 0;
}

int fnb_evolver_evaluate_d(fnb_evolver* ev, const float* d_X, const float* d_Y, int batch, int fitness_kind,
                           double fitness_offset) {
  return evolver_eval_enqueue(ev, 0, ev->ev.P, d_X, d_Y, batch, fitness_kind, fitness_offset, ev->ev.fitness);
}

// Synchronises the evolver stream and reports the last evaluation's errors in
// the reference's order (forward_into, network.hpp:238-268 via transform,
// network.hpp:122-220): the lowest genome whose transform failed, with the
// reference's message, else a non-finite input.
int fnb_evolver_eval_check(fnb_evolver* ev) {
  fnb::Evolver& v = ev->ev;
  fnb_ctx* ctx = ev->ctx;
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  ctx->err_index = -1;
  if (!ev->eflags.p) return 0;
  int fl[2] = {INT_MAX, 0};
  EV_CK(cudaMemcpyAsync(fl, ev->eflags.p, sizeof(fl), cudaMemcpyDeviceToHost, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  if (fl[0] != INT_MAX) {
    const int lo = ev->eval_lo;
    const int st = fnb_check_nets_d(ctx, v.pn[v.cur] + size_t(lo) * v.gn(), v.pc[v.cur] + size_t(lo) * v.gc(),
                                    ev->nets.p, ev->eval_n, v.st);
    if (st && ctx->err_index >= 0) ctx->err_index += lo;
    if (st) return st;
  }
  if (fl[1]) return fnb_set_error(ctx, FNB_E_NON_FINITE_INPUT, "input not finite", 0);
  return 0;
}

// host-data variant: inputs / targets as FP64 host arrays (B x I, B x O)
int fnb_evolver_evaluate(fnb_evolver* ev, const double* X, const double* Y, int batch, int fitness_kind,
                         double fitness_offset) {
  fnb::Evolver& v = ev->ev;
  fnb_ctx* ctx = ev->ctx;
  cudaSetDevice(ctx->device);
  const size_t nx = size_t(batch) * ctx->sh.I, ny = size_t(batch) * ctx->sh.O;
  if (batch <= 0) return fnb_set_error(ctx, FNB_E_EMPTY_DATASET, "batch is empty", -1);
  std::vector<float> xf(nx), yf(ny);
  for (size_t i = 0; i < nx; ++i) {
    if (!std::isfinite(X[i])) return fnb_set_error(ctx, FNB_E_NON_FINITE_INPUT, "input not finite", 0);
    xf[i] = float(X[i]);
  }
  for (size_t i = 0; i < ny; ++i) yf[i] = float(Y[i]);
  EV_CK(ev->X.ensure(sizeof(float) * nx + 16));
  EV_CK(ev->Y.ensure(sizeof(float) * ny + 16));
  EV_CK(cudaMemcpyAsync(ev->X.p, xf.data(), sizeof(float) * nx, cudaMemcpyHostToDevice, v.st));
  EV_CK(cudaMemcpyAsync(ev->Y.p, yf.data(), sizeof(float) * ny, cudaMemcpyHostToDevice, v.st));
  int st = fnb_evolver_evaluate_d(ev, static_cast<float*>(ev->X.p), static_cast<float*>(ev->Y.p), batch,
                                  fitness_kind, fitness_offset);
  if (st) return st;
  return fnb_evolver_eval_check(ev);
}

int fnb_evolver_step(fnb_evolver* ev) {
  cudaSetDevice(ev->ctx->device);
  int err = -1;
  EV_CK(ev->ev.step(&err));
  if (err == -2) return fnb_set_error(ev->ctx, FNB_E_EVAL_ERROR, "spawn counts do not sum to pop_size", -1);
  if (err >= 0) return fnb_set_error(ev->ctx, FNB_E_DUPLICATE_KEY, "mutation failed in child slot", err);
  return 0;
}

int fnb_evolver_validate(fnb_evolver* ev, int* first_invalid) {
  fnb::Evolver& v = ev->ev;
  cudaSetDevice(ev->ctx->device);
  fnb_ctx* ctx = ev->ctx;
  EV_CK(ctx->misc.ensure(sizeof(int32_t) * 2 * size_t(v.P)));
  int32_t* codes = static_cast<int32_t*>(ctx->misc.p);
  EV_CK(fnb::launch_validate(v.pn[v.cur], v.pc[v.cur], v.P, v.sh, codes, codes + v.P, v.st));
  ++ctx->launches;
  std::vector<int32_t> h(2 * size_t(v.P));
  EV_CK(cudaMemcpyAsync(h.data(), codes, sizeof(int32_t) * 2 * size_t(v.P), cudaMemcpyDeviceToHost, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  int bad = -1;
  for (int p = 0; p < v.P && bad < 0; ++p)
    if (h[p]) bad = p;
  if (first_invalid) *first_invalid = bad;
  if (bad >= 0) return fnb_set_error(ctx, FNB_E_CORRUPT_ROW, fnb::validate_message(h[bad], h[v.P + bad]), bad);
  return 0;
}

int fnb_evolver_step_front(fnb_evolver* ev) {
  cudaSetDevice(ev->ctx->device);
  EV_CK(ev->ev.front_eager());
  return 0;
}

int fnb_evolver_step_back(fnb_evolver* ev, int lo, int hi) {
  if (lo < 0 || hi > ev->ev.P || lo > hi) return fnb_set_error(ev->ctx, FNB_E_CONFIG_ERROR, "slot range out of bounds", -1);
  cudaSetDevice(ev->ctx->device);
  EV_CK(ev->ev.back_eager(lo, hi));
  return 0;
}

int fnb_evolver_step_commit(fnb_evolver* ev) {
  cudaSetDevice(ev->ctx->device);
  int err = -1;
  EV_CK(ev->ev.commit(&err));
  if (err == -2) return fnb_set_error(ev->ctx, FNB_E_EVAL_ERROR, "spawn counts do not sum to pop_size", -1);
  if (err >= 0) return fnb_set_error(ev->ctx, FNB_E_DUPLICATE_KEY, "mutation failed in child slot", err);
  return 0;
}

int fnb_evolver_next_population(fnb_evolver* ev, double** d_nodes, double** d_conns) {
  fnb::Evolver& v = ev->ev;
  if (d_nodes) *d_nodes = v.pn[v.cur ^ 1];
  if (d_conns) *d_conns = v.pc[v.cur ^ 1];
  return 0;
}

int fnb_evolver_species(fnb_evolver* ev, int* count, int* ids, int* sizes, int* spawn, double* best, int* stagnation,
                        int* species_of) {
  fnb::Evolver& v = ev->ev;
  cudaSetDevice(ev->ctx->device);
  fnb::SpeciesDev h;
  EV_CK(cudaMemcpyAsync(&h, v.sd, sizeof(h), cudaMemcpyDeviceToHost, v.st));
  if (species_of) EV_CK(cudaMemcpyAsync(species_of, v.species_of, sizeof(int) * v.P, cudaMemcpyDeviceToHost, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  if (count) *count = h.count;
  for (int j = 0; j < h.count; ++j) {
    if (ids) ids[j] = h.id[j];
    if (sizes) sizes[j] = h.size[j];
    if (spawn) spawn[j] = h.spawn[j];
    if (best) best[j] = h.best[j];
    if (stagnation) stagnation[j] = h.stag[j];
  }
  return 0;
}

int fnb_evolver_state(fnb_evolver* ev, int* generation, int* next_key) {
  fnb::Evolver& v = ev->ev;
  cudaSetDevice(ev->ctx->device);
  int nk[2] = {0, 0};
  EV_CK(cudaMemcpyAsync(nk, v.next_key, sizeof(nk), cudaMemcpyDeviceToHost, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  if (generation) *generation = v.generation;
  if (next_key) *next_key = nk[0];
  return 0;
}

// evaluate genomes [lo, hi) only, writing d_fitness_out[0 .. hi-lo) (a rank's
// shard of the population in the multi-GPU loop)
int fnb_evolver_evaluate_range_d(fnb_evolver* ev, int lo, int hi, const float* d_X, const float* d_Y, int batch,
                                 int fitness_kind, double fitness_offset, double* d_fitness_out) {
  if (lo < 0 || hi > ev->ev.P || lo > hi) return fnb_set_error(ev->ctx, FNB_E_SHAPE_MISMATCH, "bad genome range", -1);
  return evolver_eval_enqueue(ev, lo, hi - lo, d_X, d_Y, batch, fitness_kind, fitness_offset, d_fitness_out);
}

// population checksum: sum over 64-bit words w_i * (2i + 1) mod 2^64 (order
// independent, so deterministic under atomics); replicas compare it
__global__ void k_checksum(const unsigned long long* __restrict__ a, size_t n, size_t base,
                           unsigned long long* out) {
  unsigned long long s = 0;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    s += a[i] * (2ull * (base + i) + 1ull);
  for (int d = 16; d > 0; d >>= 1) s += __shfl_down_sync(0xffffffffu, s, d);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

int fnb_evolver_checksum(fnb_evolver* ev, uint64_t* out) {
  fnb::Evolver& v = ev->ev;
  fnb_ctx* ctx = ev->ctx;
  cudaSetDevice(ctx->device);
  EV_CK(ctx->partial.ensure(16));
  unsigned long long* d = static_cast<unsigned long long*>(ctx->partial.p);
  EV_CK(cudaMemsetAsync(d, 0, 8, v.st));
  const size_t nn = v.gn() * v.P, nc = v.gc() * v.P;
  k_checksum<<<4 * 148, 256, 0, v.st>>>(reinterpret_cast<const unsigned long long*>(v.pn[v.cur]), nn, 0, d);
  k_checksum<<<4 * 148, 256, 0, v.st>>>(reinterpret_cast<const unsigned long long*>(v.pc[v.cur]), nc, nn, d);
  ctx->launches += 2;
  uint64_t h = 0;
  int nk = 0;
  EV_CK(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, v.st));
  EV_CK(cudaMemcpyAsync(&nk, v.next_key, sizeof(int), cudaMemcpyDeviceToHost, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  *out = h ^ (uint64_t(uint32_t(nk)) << 32) ^ uint64_t(uint32_t(v.generation));
  return 0;
}

// device-to-device fitness injection on the evolver stream (after a gather)
int fnb_evolver_set_fitness_d(fnb_evolver* ev, const double* d_fitness) {
  fnb::Evolver& v = ev->ev;
  cudaSetDevice(ev->ctx->device);
  EV_CK(cudaMemcpyAsync(v.fitness, d_fitness, sizeof(double) * v.P, cudaMemcpyDeviceToDevice, v.st));
  return 0;
}

int fnb_evolver_set_next_key(fnb_evolver* ev, int next_key) {
  fnb::Evolver& v = ev->ev;
  cudaSetDevice(ev->ctx->device);
  const int nk[2] = {next_key, 0};
  EV_CK(cudaMemcpyAsync(v.next_key, nk, sizeof(nk), cudaMemcpyHostToDevice, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  return 0;
}

int fnb_evolver_device_state(fnb_evolver* ev, double** d_nodes, double** d_conns, double** d_fitness,
                             void** stream) {
  fnb::Evolver& v = ev->ev;
  if (d_nodes) *d_nodes = v.pn[v.cur];
  if (d_conns) *d_conns = v.pc[v.cur];
  if (d_fitness) *d_fitness = v.fitness;
  if (stream) *stream = v.st;
  return 0;
}

}  // extern "C"

// =================================================================================
// checkpoint / resume (SPEC.md:337-340 SpeciesState, :122 / :525-532 save-load):
// everything a generation step reads besides the population -- the seed (the
// key tree, oracle E1), the generation counter, the InnovationTable counter,
// and the species table with its representatives.
// =================================================================================
extern "C" {

int fnb_evolver_get_state(fnb_evolver* ev, fnb_run_state* s, double* rep_nodes, double* rep_conns) {
  fnb::Evolver& v = ev->ev;
  if (!s) return fnb_set_error(ev->ctx, FNB_E_CONFIG_ERROR, "no state buffer", -1);
  cudaSetDevice(ev->ctx->device);
  fnb::SpeciesDev h;
  int nk[2] = {0, 0};
  EV_CK(cudaMemcpyAsync(&h, v.sd, sizeof(h), cudaMemcpyDeviceToHost, v.st));
  EV_CK(cudaMemcpyAsync(nk, v.next_key, sizeof(nk), cudaMemcpyDeviceToHost, v.st));
  if (rep_nodes && h.count > 0)
    EV_CK(cudaMemcpyAsync(rep_nodes, v.rep_n, sizeof(double) * v.gn() * h.count, cudaMemcpyDeviceToHost, v.st));
  if (rep_conns && h.count > 0)
    EV_CK(cudaMemcpyAsync(rep_conns, v.rep_c, sizeof(double) * v.gc() * h.count, cudaMemcpyDeviceToHost, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  *s = fnb_run_state{};
  s->seed = v.seed;
  s->generation = v.generation;
  s->next_key = nk[0];
  s->species_count = h.count;
  s->next_species_id = h.next_id;
  for (int j = 0; j < h.count; ++j) {
    s->species_id[j] = h.id[j];
    s->species_best[j] = h.best[j];
    s->species_stagnation[j] = h.stag[j];
    s->species_size[j] = h.size[j];
    s->species_spawn[j] = h.spawn[j];
  }
  return 0;
}

int fnb_evolver_set_state(fnb_evolver* ev, const fnb_run_state* s, const double* rep_nodes, const double* rep_conns) {
  fnb::Evolver& v = ev->ev;
  fnb_ctx* ctx = ev->ctx;
  if (!s || s->species_count < 0 || s->species_count > v.cfg.max_species || s->generation < 0 ||
      (s->species_count > 0 && (!rep_nodes || !rep_conns)))
    return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "invalid evolver state", -1);
  for (int j = 0; j < s->species_count; ++j)
    if (s->species_id[j] < 0 || s->species_id[j] >= s->next_species_id || (j && s->species_id[j] <= s->species_id[j - 1]))
      return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "species ids must ascend below next_species_id", j);
  cudaSetDevice(ctx->device);
  fnb::SpeciesDev h{};
  h.count = s->species_count;
  h.next_id = s->next_species_id;
  h.generation = s->generation;
  h.first_bad = INT_MAX;
  for (int j = 0; j < s->species_count; ++j) {
    h.id[j] = s->species_id[j];
    h.best[j] = s->species_best[j];
    h.stag[j] = s->species_stagnation[j];
    h.size[j] = s->species_size[j];
    h.spawn[j] = s->species_spawn[j];
  }
  const int nk[2] = {s->next_key, 0};
  EV_CK(cudaMemcpyAsync(v.sd, &h, sizeof(h), cudaMemcpyHostToDevice, v.st));
  EV_CK(cudaMemcpyAsync(v.next_key, nk, sizeof(nk), cudaMemcpyHostToDevice, v.st));
  if (s->species_count > 0) {
    EV_CK(cudaMemcpyAsync(v.rep_n, rep_nodes, sizeof(double) * v.gn() * s->species_count, cudaMemcpyHostToDevice,
                          v.st));
    EV_CK(cudaMemcpyAsync(v.rep_c, rep_conns, sizeof(double) * v.gc() * s->species_count, cudaMemcpyHostToDevice,
                          v.st));
  }
  EV_CK(cudaStreamSynchronize(v.st));
  v.seed = s->seed;
  v.generation = s->generation;
  v.host_species = s->species_count;
  return 0;
}

}  // extern "C"

// =================================================================================
// SPEC evolve(problem, cfg, key) (PAPER Algorithm 1) as one
// device-resident loop.  Each generation is ONE CUDA graph:
//     K1 + K2 (evaluate) -> k_gen_stats -> IF (no error and best < target) { step }
// The conditional node (cudaGraphCondTypeIf, set from k_gen_stats) keeps the
// termination check BEFORE reproduction without a host round
// trip between evaluation and the step; the host reads one small GenStats
// record per generation for RunStats.  Graphs are keyed like the step graphs
// by (species count before the step, current buffer).  Without conditional
// node support the same sequence runs as an evaluate graph, a host check and
// the step graph.
// =================================================================================
namespace fnb {

struct GenStats {
  double best, mean, std;
  int best_index;
  int eval_first_bad;   // lowest genome whose transform failed (INT_MAX none)
  int eval_nonfinite;
  int stepped;          // the step body ran
  int step_error, species_count, first_bad;
  int species_size[kMaxSpecies];
};

// Fitness statistics in one CTA, in a fixed order (deterministic for a given
// P): each thread reduces a contiguous run, then a fixed shared-memory tree.
// best = max (lowest index on ties), mean = sum / P, std = population std.
__global__ void __launch_bounds__(1024) k_gen_stats(const double* __restrict__ fit, int P, const int* eflags,
                                                    double target, cudaGraphConditionalHandle h, int use_cond,
                                                    GenStats* out) {
  __shared__ double s_sum[1024];
  __shared__ double s_max[1024];
  __shared__ int s_arg[1024];
  __shared__ double s_mean;
  const int t = threadIdx.x, nt = blockDim.x;
  const int per = (P + nt - 1) / nt, lo = min(P, t * per), hi = min(P, lo + per);
  double sum = 0.0, mx = -INFINITY;
  int arg = INT_MAX;
  for (int i = lo; i < hi; ++i) {
    const double f = fit[i];
    sum = __dadd_rn(sum, f);
    if (arg == INT_MAX || f > mx) { mx = f; arg = i; }
  }
  s_sum[t] = sum;
  s_max[t] = mx;
  s_arg[t] = arg;
  __syncthreads();
  for (int d = nt / 2; d > 0; d >>= 1) {
    if (t < d) {
      s_sum[t] = __dadd_rn(s_sum[t], s_sum[t + d]);
      const bool take = s_arg[t + d] != INT_MAX &&
                        (s_arg[t] == INT_MAX || s_max[t + d] > s_max[t] ||
                         (s_max[t + d] == s_max[t] && s_arg[t + d] < s_arg[t]));
      if (take) { s_max[t] = s_max[t + d]; s_arg[t] = s_arg[t + d]; }
    }
    __syncthreads();
  }
  if (t == 0) s_mean = __ddiv_rn(s_sum[0], double(P));
  __syncthreads();
  const double mean = s_mean;
  double sq = 0.0;
  for (int i = lo; i < hi; ++i) {
    const double d = __dsub_rn(fit[i], mean);
    sq = __dadd_rn(sq, __dmul_rn(d, d));
  }
  __syncthreads();
  s_sum[t] = sq;
  __syncthreads();
  for (int d = nt / 2; d > 0; d >>= 1) {
    if (t < d) s_sum[t] = __dadd_rn(s_sum[t], s_sum[t + d]);
    __syncthreads();
  }
  if (t == 0) {
    out->best = s_max[0];
    out->best_index = s_arg[0];
    out->mean = mean;
    out->std = sqrt(__ddiv_rn(s_sum[0], double(P)));
    out->eval_first_bad = eflags[0];
    out->eval_nonfinite = eflags[1];
    out->stepped = 0;
    const bool ok = eflags[0] == INT_MAX && eflags[1] == 0;
    const bool done = s_max[0] >= target;
    if (use_cond) cudaGraphSetConditional(h, ok && !done ? 1u : 0u);
  }
}

// the step's outcome for the host (tail of the conditional body)
__global__ void k_gen_step_status(const SpeciesDev* sd, GenStats* out) {
  const int t = threadIdx.x;
  if (t < kMaxSpecies) out->species_size[t] = t < sd->count ? sd->size[t] : 0;
  if (t == 0) {
    out->stepped = 1;
    out->step_error = sd->error;
    out->species_count = sd->count;
    out->first_bad = sd->first_bad;
  }
}

}  // namespace fnb

struct fnb_gen_graph {
  cudaGraphExec_t exec = nullptr;
  long long n_eval = 0, n_step = 0;
};

// The graphs bake in the problem (device X / Y, batch, fitness kind and
// offset, target), so they are kept across fnb_evolve calls with the same key.
struct fnb_evolve_run {
  fnb_gen_graph g[fnb::kMaxSpecies + 1][2];
  bool use_cond = true;
  fnb::GenStats* d_stats = nullptr;
  fnb::GenStats* h_stats = nullptr;  // pinned
  const void* key_x = nullptr;
  const void* key_y = nullptr;
  const void* key_bufs[3] = {nullptr, nullptr, nullptr};  // partial sums, nets, eval flags
  int key_batch = -1, key_kind = -1;
  double key_offset = 0.0, key_target = 0.0;
  void drop_graphs() {
    for (auto& row : g)
      for (auto& x : row)
        if (x.exec) {
          cudaGraphExecDestroy(x.exec);
          x.exec = nullptr;
        }
  }
  ~fnb_evolve_run() {
    drop_graphs();
    if (d_stats) cudaFree(d_stats);
    if (h_stats) cudaFreeHost(h_stats);
  }
};

static void release_evolve_run(fnb_evolve_run* r) { delete r; }

static long long count_kernel_nodes(cudaGraph_t graph) {
  size_t n = 0;
  if (cudaGraphGetNodes(graph, nullptr, &n) != cudaSuccess || n == 0) return 0;
  std::vector<cudaGraphNode_t> nodes(n);
  if (cudaGraphGetNodes(graph, nodes.data(), &n) != cudaSuccess) return 0;
  long long k = 0;
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

// evaluate + stats (+ the conditional step when `with_step`) for the current
// (species count, buffer), captured on the evolver stream.
static cudaError_t build_gen_graph(fnb_evolver* ev, fnb_evolve_run& run, const float* X, const float* Y, int batch,
                                   int kind, double offset, double target, fnb_gen_graph* out) {
  fnb::Evolver& v = ev->ev;
  fnb_ctx* ctx = ev->ctx;
  const long long before = ctx->launches;
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamBeginCapture(v.st, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return e;
  cudaGraphConditionalHandle h = 0;
  cudaStreamCaptureStatus cs;
  cudaGraph_t cap = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  e = cudaStreamGetCaptureInfo(v.st, &cs, nullptr, &cap, nullptr, nullptr);
  if (e == cudaSuccess && run.use_cond) e = cudaGraphConditionalHandleCreate(&h, cap, 0, cudaGraphCondAssignDefault);
  int st = 0;
  if (e == cudaSuccess) st = evolver_eval_enqueue(ev, 0, v.P, X, Y, batch, kind, offset, v.fitness);
  if (e == cudaSuccess && !st) {
    fnb::k_gen_stats<<<1, 1024, 0, v.st>>>(v.fitness, v.P, static_cast<const int*>(ev->eflags.p), target, h,
                                            run.use_cond ? 1 : 0, run.d_stats);
    e = cudaGetLastError();
  }
  cudaGraphNode_t cond = nullptr;
  cudaGraph_t body = nullptr;
  if (e == cudaSuccess && !st && run.use_cond) {
    e = cudaStreamGetCaptureInfo(v.st, &cs, nullptr, &cap, &deps, &ndeps);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeIf;
    p.conditional.size = 1;
    if (e == cudaSuccess) e = cudaGraphAddNode(&cond, cap, deps, ndeps, &p);
    if (e == cudaSuccess) {
      body = p.conditional.phGraph_out[0];
      e = cudaStreamUpdateCaptureDependencies(v.st, &cond, 1, cudaStreamSetCaptureDependencies);
    }
  }
  const cudaError_t ee = cudaStreamEndCapture(v.st, &graph);
  if (e == cudaSuccess) e = ee;
  if (st && e == cudaSuccess) e = cudaErrorInvalidValue;
  const long long n_eval = ctx->launches - before + 1;
  long long n_step = 0;
  if (e == cudaSuccess && body) {  // the step, captured into the conditional body
    const long long b2 = ctx->launches;
    e = cudaStreamBeginCaptureToGraph(v.st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      cudaError_t es = v.enqueue_step();
      if (es == cudaSuccess) {
        fnb::k_gen_step_status<<<1, 32, 0, v.st>>>(v.sd, run.d_stats);
        es = cudaGetLastError();
      }
      cudaGraph_t b_out = nullptr;
      e = cudaStreamEndCapture(v.st, &b_out);
      if (es != cudaSuccess) e = es;
    }
    n_step = ctx->launches - b2 + 1;
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&out->exec, graph, 0);
  if (e == cudaSuccess) {
    out->n_eval = run.use_cond ? n_eval : count_kernel_nodes(graph);
    out->n_step = n_step;
  }
  if (graph) cudaGraphDestroy(graph);
  ctx->launches = before;
  return e;
}

extern "C" {

int fnb_evolve(fnb_evolver* ev, const double* inputs, const double* targets, int batch, int fitness_kind,
               double fitness_offset, double fitness_target, int generation_limit, fnb_run_stats_fn on_generation,
               void* user, double* best_nodes, double* best_conns, double* best_fitness, int* generations_run) {
  fnb::Evolver& v = ev->ev;
  fnb_ctx* ctx = ev->ctx;
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  ctx->err_index = -1;
  if (generations_run) *generations_run = 0;
  if (batch <= 0) return fnb_set_error(ctx, FNB_E_EMPTY_DATASET, "batch is empty", -1);
  if (generation_limit < 0 || fitness_kind == FNB_FIT_NONE)
    return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "generation_limit >= 0 and a fitness kind are required", -1);
  // the problem's data go up once, narrowed to FP32 (the forward's arithmetic)
  const size_t nx = size_t(batch) * ctx->sh.I, ny = size_t(batch) * ctx->sh.O;
  std::vector<float> xf(nx), yf(ny);
  for (size_t i = 0; i < nx; ++i) {
    if (!std::isfinite(inputs[i])) return fnb_set_error(ctx, FNB_E_NON_FINITE_INPUT, "input not finite", 0);
    xf[i] = float(inputs[i]);
  }
  for (size_t i = 0; i < ny; ++i) yf[i] = float(targets[i]);
  EV_CK(ev->X.ensure(sizeof(float) * nx + 16));
  EV_CK(ev->Y.ensure(sizeof(float) * ny + 16));
  EV_CK(cudaMemcpyAsync(ev->X.p, xf.data(), sizeof(float) * nx, cudaMemcpyHostToDevice, v.st));
  EV_CK(cudaMemcpyAsync(ev->Y.p, yf.data(), sizeof(float) * ny, cudaMemcpyHostToDevice, v.st));
  EV_CK(ev->nets.ensure(ctx->L.bytes * size_t(v.P)));
  EV_CK(ev->eflags.ensure(4 * sizeof(int)));
  EV_CK(ctx->partial.ensure(fnb::forward_partial_needed(ctx->L, v.P, batch)));
  const float* X = static_cast<const float*>(ev->X.p);
  const float* Y = static_cast<const float*>(ev->Y.p);
  if (!ev->run) ev->run = new fnb_evolve_run();
  fnb_evolve_run& run = *ev->run;
  if (!run.d_stats) EV_CK(cudaMalloc(&run.d_stats, sizeof(fnb::GenStats)));
  if (!run.h_stats) EV_CK(cudaMallocHost(&run.h_stats, sizeof(fnb::GenStats)));
  EV_CK(cudaStreamSynchronize(v.st));
  bool use_graphs = v.use_graphs;
  bool want_cond = true;
  if (const char* g = std::getenv("FNB_GEN_GRAPH")) want_cond = std::string(g) != "0";
  if (run.key_x != X || run.key_y != Y || run.key_batch != batch || run.key_kind != fitness_kind ||
      run.key_offset != fitness_offset || run.key_target != fitness_target || run.use_cond != want_cond ||
      run.key_bufs[0] != ctx->partial.p || run.key_bufs[1] != ev->nets.p || run.key_bufs[2] != ev->eflags.p) {
    run.drop_graphs();  // another problem (or mode): the cached graphs do not apply
    run.use_cond = want_cond;
    run.key_x = X;
    run.key_y = Y;
    run.key_batch = batch;
    run.key_kind = fitness_kind;
    run.key_offset = fitness_offset;
    run.key_target = fitness_target;
    run.key_bufs[0] = ctx->partial.p;
    run.key_bufs[1] = ev->nets.p;
    run.key_bufs[2] = ev->eflags.p;
  }
  int last_eval_buf = v.cur, last_best = 0;
  double last_fit = -INFINITY;
  int gens = 0;
  for (int g = 0; g < generation_limit; ++g) {
    const auto t0 = std::chrono::steady_clock::now();
    const int eval_buf = v.cur, gen_no = v.generation;
    bool stepped_in_graph = false;
    fnb_gen_graph* gg = nullptr;
    if (use_graphs) {
      gg = &run.g[v.host_species][v.cur];
      if (!gg->exec) {
        cudaError_t e = build_gen_graph(ev, run, X, Y, batch, fitness_kind, fitness_offset, fitness_target, gg);
        if (e != cudaSuccess && run.use_cond) {  // no conditional nodes here: evaluate graph + host check
          cudaGetLastError();
          run.use_cond = false;
          run.drop_graphs();
          e = build_gen_graph(ev, run, X, Y, batch, fitness_kind, fitness_offset, fitness_target, gg);
        }
        if (e != cudaSuccess) {
          cudaGetLastError();
          use_graphs = false;
          gg = nullptr;
        }
      }
    }
    if (gg) {
      EV_CK(cudaGraphLaunch(gg->exec, v.st));
      ctx->launches += gg->n_eval;
    } else {
      if (int st = evolver_eval_enqueue(ev, 0, v.P, X, Y, batch, fitness_kind, fitness_offset, v.fitness)) return st;
      fnb::k_gen_stats<<<1, 1024, 0, v.st>>>(v.fitness, v.P, static_cast<const int*>(ev->eflags.p), fitness_target,
                                              0, 0, run.d_stats);
      EV_CK(cudaGetLastError());
      ++ctx->launches;
    }
    EV_CK(cudaMemcpyAsync(run.h_stats, run.d_stats, sizeof(fnb::GenStats), cudaMemcpyDeviceToHost, v.st));
    EV_CK(cudaStreamSynchronize(v.st));
    const fnb::GenStats s = *run.h_stats;
    if (s.eval_first_bad != INT_MAX || s.eval_nonfinite) {  // abort with context
      ev->eval_lo = 0;
      ev->eval_n = v.P;
      int st = 0;
      if (s.eval_first_bad != INT_MAX)
        st = fnb_check_nets_d(ctx, v.pn[eval_buf], v.pc[eval_buf], ev->nets.p, v.P, v.st);
      if (!st) st = fnb_set_error(ctx, FNB_E_NON_FINITE_INPUT, "input not finite", 0);
      ctx->err = ctx->err.substr(0, ctx->err.find(": ") + 2) + "generation " + std::to_string(gen_no) + ", genome " +
                 std::to_string(ctx->err_index) + ": " + ctx->err.substr(ctx->err.find(": ") + 2);
      return st;
    }
    const bool done = s.best >= fitness_target;
    fnb_run_stats rs{};
    rs.generation = gen_no;
    rs.best = s.best;
    rs.mean = s.mean;
    rs.std = s.std;
    rs.best_index = s.best_index;
    if (gg && run.use_cond) {
      stepped_in_graph = s.stepped != 0;
      if (stepped_in_graph) {
        ctx->launches += gg->n_step;
        if (s.step_error) return fnb_set_error(ctx, FNB_E_EVAL_ERROR, "spawn counts do not sum to pop_size", -1);
        if (s.first_bad != INT_MAX)
          return fnb_set_error(ctx, FNB_E_DUPLICATE_KEY, "mutation failed in child slot", s.first_bad);
        v.host_species = s.species_count;
        v.cur ^= 1;
        ++v.generation;
      }
    } else if (!done) {
      int err = -1;
      EV_CK(v.step(&err));
      if (err == -2) return fnb_set_error(ctx, FNB_E_EVAL_ERROR, "spawn counts do not sum to pop_size", -1);
      if (err >= 0) return fnb_set_error(ctx, FNB_E_DUPLICATE_KEY, "mutation failed in child slot", err);
    }
    // species after this generation's speciation (the previous table when it stopped first)
    fnb::SpeciesDev h;
    if (!stepped_in_graph) {
      EV_CK(cudaMemcpyAsync(&h, v.sd, sizeof(h), cudaMemcpyDeviceToHost, v.st));
      EV_CK(cudaStreamSynchronize(v.st));
      rs.species_count = h.count;
      for (int j = 0; j < h.count; ++j) rs.species_size[j] = h.size[j];
    } else {
      rs.species_count = s.species_count;
      for (int j = 0; j < s.species_count; ++j) rs.species_size[j] = s.species_size[j];
    }
    rs.elapsed_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    last_eval_buf = eval_buf;
    last_best = s.best_index;
    last_fit = s.best;
    ++gens;
    const int stop = on_generation ? on_generation(user, &rs) : 0;
    if (done || stop) break;
  }
  if (generations_run) *generations_run = gens;
  if (best_fitness) *best_fitness = last_fit;
  ev->run_mode = use_graphs ? (run.use_cond ? 2 : 1) : 0;
  // pop[argmax(fit)] of the last evaluated generation: one genome leaves the device
  if (gens > 0 && best_nodes)
    EV_CK(cudaMemcpyAsync(best_nodes, v.pn[last_eval_buf] + size_t(last_best) * v.gn(), sizeof(double) * v.gn(),
                          cudaMemcpyDeviceToHost, v.st));
  if (gens > 0 && best_conns)
    EV_CK(cudaMemcpyAsync(best_conns, v.pc[last_eval_buf] + size_t(last_best) * v.gc(), sizeof(double) * v.gc(),
                          cudaMemcpyDeviceToHost, v.st));
  EV_CK(cudaStreamSynchronize(v.st));
  return 0;
}

}  // extern "C"

extern "C" int fnb_evolver_run_mode(fnb_evolver* ev) { return ev ? ev->run_mode : -1; }

// =================================================================================
// the step sharded over ranks: phases and the buffers the caller's collectives
// reduce between them (include/flatneat_b200.h, distributed.py ShardedEvolution)
// =================================================================================
extern "C" {

int fnb_evolver_host_species(fnb_evolver* ev) { return ev ? ev->ev.host_species : -1; }

int fnb_evolver_shard_init(fnb_evolver* ev, int world, const int* bounds) {
  fnb::Evolver& v = ev->ev;
  if (world < 1 || !bounds || bounds[0] != 0 || bounds[world] != v.P)
    return fnb_set_error(ev->ctx, FNB_E_CONFIG_ERROR, "shard bounds must split [0, pop_size)", -1);
  for (int r = 0; r < world; ++r)
    if (bounds[r + 1] < bounds[r]) return fnb_set_error(ev->ctx, FNB_E_CONFIG_ERROR, "shard bounds must ascend", r);
  cudaSetDevice(ev->ctx->device);
  EV_CK(v.shard_init(world, bounds));
  return 0;
}

int fnb_evolver_shard_buffers(fnb_evolver* ev, fnb_shard_buffers* b) {
  fnb::Evolver& v = ev->ev;
  if (!b || !v.need) return fnb_set_error(ev->ctx, FNB_E_CONFIG_ERROR, "fnb_evolver_shard_init first", -1);
  uint8_t* sd = reinterpret_cast<uint8_t*>(v.sd);
  *b = fnb_shard_buffers{};
  b->min_unassigned = v.min_u;
  b->rep_dmin = reinterpret_cast<unsigned long long*>(sd + offsetof(fnb::SpeciesDev, dmin));
  b->rep_argmin = reinterpret_cast<int*>(sd + offsetof(fnb::SpeciesDev, argmin));
  b->rep_stage = v.stage;
  b->rep_stage_words = (v.gn() + v.gc()) * fnb::kMaxSpecies;
  b->species_size = reinterpret_cast<int*>(sd + offsetof(fnb::SpeciesDev, size));
  b->species_max = reinterpret_cast<unsigned long long*>(sd + offsetof(fnb::SpeciesDev, mxbits));
  b->rank_sum = reinterpret_cast<long long*>(sd + offsetof(fnb::SpeciesDev, rsum));
  b->rank_count = reinterpret_cast<int*>(sd + offsetof(fnb::SpeciesDev, cnt));
  b->first_bad = reinterpret_cast<int*>(sd + offsetof(fnb::SpeciesDev, first_bad));
  b->fitness = v.fitness;
  b->species_of = v.species_of;
  b->rep_nodes = v.rep_n;
  b->rep_conns = v.rep_c;
  b->send_nodes = v.send_n;
  b->send_conns = v.send_c;
  b->pool_nodes = v.pool_n;
  b->pool_conns = v.pool_c;
  return 0;
}

int fnb_evolver_shard_phase(fnb_evolver* ev, int phase, int rank, int a, int b, int* out) {
  fnb::Evolver& v = ev->ev;
  fnb_ctx* ctx = ev->ctx;
  if (!v.need || rank < 0 || rank >= v.sh_world)
    return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "fnb_evolver_shard_init first / rank out of range", -1);
  cudaSetDevice(ctx->device);
  const int lo = v.sh_bounds[size_t(rank)], hi = v.sh_bounds[size_t(rank) + 1];
  switch (phase) {
    case FNB_SHARD_BEGIN: EV_CK(v.shard_begin(lo, hi)); break;
    case FNB_SHARD_MIN_UNASSIGNED: EV_CK(v.shard_min_unassigned(lo, hi)); break;
    case FNB_SHARD_FOUND:
      if (a < 0 || a >= v.P || b < 0 || b >= v.cfg.max_species)
        return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "founder / species slot out of range", a);
      if (a >= lo && a < hi) EV_CK(v.shard_found(a, b));
      break;
    case FNB_SHARD_JOIN:
      if (b < 0 || b >= v.cfg.max_species) return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "species slot out of range", b);
      EV_CK(v.shard_join(lo, hi, b));
      break;
    case FNB_SHARD_ASSIGN_REST: EV_CK(v.shard_assign_rest(lo, hi)); break;
    case FNB_SHARD_REP_ARGMIN: EV_CK(v.shard_rep_argmin(lo, hi)); break;
    case FNB_SHARD_REP_STAGE: EV_CK(v.shard_rep_stage(lo, hi)); break;
    case FNB_SHARD_REP_COMMIT: EV_CK(v.shard_rep_commit(lo, hi)); break;
    case FNB_SHARD_COMPACT: EV_CK(v.shard_compact(lo, hi)); break;
    case FNB_SHARD_STAGNATION: EV_CK(v.shard_stagnation(lo, hi)); break;
    case FNB_SHARD_SELECT: {
      EV_CK(v.shard_select());
      if (out) {
        EV_CK(cudaMemcpyAsync(out, v.counts, sizeof(int) * size_t(v.sh_world), cudaMemcpyDeviceToHost, v.st));
        EV_CK(cudaStreamSynchronize(v.st));
      }
      break;
    }
    case FNB_SHARD_PACK: EV_CK(v.shard_pack(lo, hi, a)); break;
    case FNB_SHARD_BACK: EV_CK(v.shard_back(lo, hi, a)); break;
    default: return fnb_set_error(ctx, FNB_E_CONFIG_ERROR, "unknown shard phase", phase);
  }
  return 0;
}

}  // extern "C"
