/*
 * evolution.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Restatement of the SPEC-only evolution module.  The
 * reference ships NO code for these stages ("parity unpinned", SURVEY.md
 * 8c): this file freezes one precise reading of the SPEC prose, built on
 * the reference primitives restated in flatneat_oracle.c, and the CUDA
 * generation loop is held bit-exact to it.  Every choice the SPEC leaves
 * open is fixed here and listed in DESIGN.md section "Evolution semantics":
 *
 *  E1 key tree: root = RngKey(seed); init genome i = root.split(0).split(i);
 *     child slot c of generation g = root.split(1).split(g).split(c), whose
 *     split(0) drives parent selection, split(1) crossover, split(2) mutate.
 *  E2 speciate: genome i joins the first species (ascending id) whose
 *     representative r has distance(genome_i, r) < threshold (strict);
 *     unmatched genomes found species in index order while count <
 *     max_species (later genomes also test earlier founders); the rest join
 *     the nearest representative (ties: lowest id).  Old species' new rep =
 *     member closest to the old rep (ties: lowest index); founders represent
 *     new species; empty species are dropped.
 *  E3 stagnation: species max fitness > best-ever resets the counter, else
 *     +1; counter > max_stagnation removes the species unless it is among
 *     the species_elitism best (max fitness desc, ties lower id); at least
 *     one species always survives.
 *  E4 spawn: mid-rank r_i of fitness (ties share their mean position)
 *     normalised r/(P-1); species mean = exact integer sum of 2 r_i /
 *     (2 (P-1) n_j); target = P * af/sum(af); clamp to
 *     old +- round(rate*old); rescale to P; largest remainder (ties lower
 *     id); raise to genome_elitism, taking surplus from the largest
 *     allocation (ties highest id).
 *  E5 reproduce: slots laid out species by species (ascending id); members
 *     ordered (fitness desc, index asc); the first min(elitism, spawn, size)
 *     slots copy the top members; other slots draw parents a, b uniformly
 *     from the top max(1, ceil(survival*size)); fit parent = higher fitness
 *     (ties lower index); crossover then mutate with one InnovationTable
 *     assigned in slot order.
 */
#include "flatneat_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define NSZ(sh) ((size_t)(sh)->max_nodes * FO_NODE_COLS)
#define CSZ(sh) ((size_t)(sh)->max_conns * FO_CONN_COLS)

void fo_species_init(fo_species* s, const fo_shape* sh, int cap) {
  s->count = 0;
  s->next_id = 0;
  s->cap = cap;
  s->nsz = NSZ(sh);
  s->csz = CSZ(sh);
  s->id = (int*)calloc((size_t)cap, sizeof(int));
  s->rep_nodes = (double*)calloc((size_t)cap * NSZ(sh), sizeof(double));
  s->rep_conns = (double*)calloc((size_t)cap * CSZ(sh), sizeof(double));
  s->best_fitness = (double*)calloc((size_t)cap, sizeof(double));
  s->stagnation = (int*)calloc((size_t)cap, sizeof(int));
  s->size = (int*)calloc((size_t)cap, sizeof(int));
  s->spawn = (int*)calloc((size_t)cap, sizeof(int));
}

void fo_species_free(fo_species* s) {
  free(s->id); free(s->rep_nodes); free(s->rep_conns); free(s->best_fitness);
  free(s->stagnation); free(s->size); free(s->spawn);
  memset(s, 0, sizeof(*s));
}

int fo_initialize_population(const fo_shape* sh, const fo_schema* sc,
                             const fo_neat_cfg* cfg, uint64_t seed,
                             double* pop_nodes, double* pop_conns) {
  /* I inputs, O outputs, one hidden node, dense
   * input->hidden and hidden->output connections. */
  const int I = sh->num_inputs, O = sh->num_outputs;
  if (I + O + 1 > sh->max_nodes || I + O > sh->max_conns) return 1 + FO_E_limits_too_small;
  for (int i = 0; i < I; ++i) if (sh->input_keys[i] != i) return 1 + FO_E_config_error;
  for (int o = 0; o < O; ++o) if (sh->output_keys[o] != I + o) return 1 + FO_E_config_error;
  const int hidden = I + O;
  const fo_key root = fo_key_seed(seed);
  const fo_key init = fo_key_split(root, 0);
  for (int g = 0; g < cfg->pop_size; ++g) {
    double* n = pop_nodes + (size_t)g * NSZ(sh);
    double* c = pop_conns + (size_t)g * CSZ(sh);
    for (size_t k = 0; k < NSZ(sh); ++k) n[k] = NAN;
    for (size_t k = 0; k < CSZ(sh); ++k) c[k] = NAN;
    fo_stream s;
    fo_stream_init(&s, fo_key_split(init, (uint64_t)g));
    for (int i = 0; i < I; ++i) {
      double* row = n + (size_t)i * FO_NODE_COLS;
      row[0] = (double)i; row[1] = 0.0; row[2] = 1.0;
      row[3] = (double)sc->default_agg; row[4] = (double)sc->default_act;
    }
    for (int r = I; r <= hidden; ++r) {
      double* row = n + (size_t)r * FO_NODE_COLS;
      row[0] = (double)r;
      row[1] = fo_normal(&s, cfg->mutation.bias.init_mean, cfg->mutation.bias.init_std);
      row[2] = fo_normal(&s, cfg->mutation.response.init_mean, cfg->mutation.response.init_std);
      row[3] = (double)sc->default_agg;
      row[4] = (double)(r < hidden ? cfg->output_activation : sc->default_act);
    }
    for (int r = 0; r < I + O; ++r) {
      double* row = c + (size_t)r * FO_CONN_COLS;
      row[0] = (double)(r < I ? r : hidden);
      row[1] = (double)(r < I ? hidden : r);
      row[2] = 1.0;
      row[3] = fo_normal(&s, cfg->mutation.weight.init_mean, cfg->mutation.weight.init_std);
    }
  }
  return 0;
}

static void species_copy_slot(const fo_shape* sh, fo_species* s, int dst, int src) {
  if (dst == src) return;
  s->id[dst] = s->id[src];
  memcpy(s->rep_nodes + (size_t)dst * NSZ(sh), s->rep_nodes + (size_t)src * NSZ(sh), sizeof(double) * NSZ(sh));
  memcpy(s->rep_conns + (size_t)dst * CSZ(sh), s->rep_conns + (size_t)src * CSZ(sh), sizeof(double) * CSZ(sh));
  s->best_fitness[dst] = s->best_fitness[src];
  s->stagnation[dst] = s->stagnation[src];
  s->size[dst] = s->size[src];
  s->spawn[dst] = s->spawn[src];
}

void fo_speciate(const fo_shape* sh, const fo_neat_cfg* cfg, const double* pop_nodes,
                 const double* pop_conns, fo_species* s, int* species_of) {
  const int P = cfg->pop_size;
  const int S_old = s->count;
  const double th = cfg->compatibility_threshold;
  double* d_old = (double*)malloc(sizeof(double) * (size_t)P * (size_t)(S_old > 0 ? S_old : 1));
#define GN(i) (pop_nodes + (size_t)(i) * NSZ(sh))
#define GC(i) (pop_conns + (size_t)(i) * CSZ(sh))
#define RN(j) (s->rep_nodes + (size_t)(j) * NSZ(sh))
#define RC(j) (s->rep_conns + (size_t)(j) * CSZ(sh))
  for (int i = 0; i < P; ++i) {
    species_of[i] = -1;
    for (int j = 0; j < S_old; ++j) {
      const double d = fo_distance(sh, GN(i), GC(i), RN(j), RC(j), &cfg->distance);
      d_old[(size_t)i * S_old + j] = d;
      if (species_of[i] < 0 && d < th) species_of[i] = j;
    }
  }
  /* founding rounds in index order */
  for (int f = 0; f < P && s->count < cfg->max_species; ++f) {
    if (species_of[f] >= 0) continue;
    const int j = s->count++;
    s->id[j] = s->next_id++;
    memcpy(RN(j), GN(f), sizeof(double) * NSZ(sh));
    memcpy(RC(j), GC(f), sizeof(double) * CSZ(sh));
    s->best_fitness[j] = -INFINITY;
    s->stagnation[j] = 0;
    species_of[f] = j;
    for (int i = f + 1; i < P; ++i) {
      if (species_of[i] >= 0) continue;
      if (fo_distance(sh, GN(i), GC(i), GN(f), GC(f), &cfg->distance) < th) species_of[i] = j;
    }
  }
  /* overflow: nearest representative, ties -> lowest species */
  for (int i = 0; i < P; ++i) {
    if (species_of[i] >= 0) continue;
    int best = 0;
    double bd = 0.0;
    for (int j = 0; j < s->count; ++j) {
      const double d = fo_distance(sh, GN(i), GC(i), RN(j), RC(j), &cfg->distance);
      if (j == 0 || d < bd) { bd = d; best = j; }
    }
    species_of[i] = best;
  }
  /* representative update for old species: member closest to old rep */
  for (int j = 0; j < S_old; ++j) {
    int best = -1;
    double bd = 0.0;
    for (int i = 0; i < P; ++i) {
      if (species_of[i] != j) continue;
      const double d = d_old[(size_t)i * S_old + j];
      if (best < 0 || d < bd) { bd = d; best = i; }
    }
    if (best >= 0) {
      memcpy(RN(j), GN(best), sizeof(double) * NSZ(sh));
      memcpy(RC(j), GC(best), sizeof(double) * CSZ(sh));
    }
  }
  /* sizes, then drop empty species keeping id order */
  for (int j = 0; j < s->count; ++j) s->size[j] = 0;
  for (int i = 0; i < P; ++i) s->size[species_of[i]]++;
  int* remap = (int*)malloc(sizeof(int) * (size_t)(s->count > 0 ? s->count : 1));
  int k = 0;
  for (int j = 0; j < s->count; ++j) {
    if (s->size[j] == 0) { remap[j] = -1; continue; }
    remap[j] = k;
    species_copy_slot(sh, s, k, j);
    ++k;
  }
  s->count = k;
  for (int i = 0; i < P; ++i) species_of[i] = remap[species_of[i]];
  free(remap);
  free(d_old);
#undef GN
#undef GC
#undef RN
#undef RC
}

void fo_update_stagnation(const fo_neat_cfg* cfg, const double* fitness,
                          fo_species* s, int* species_of) {
  const int P = cfg->pop_size;
  const int S = s->count;
  if (S <= 0) return;
  double* mx = (double*)malloc(sizeof(double) * (size_t)S);
  int* seen = (int*)calloc((size_t)S, sizeof(int));
  for (int i = 0; i < P; ++i) {
    const int j = species_of[i];
    if (j < 0) continue;
    if (!seen[j] || fitness[i] > mx[j]) mx[j] = fitness[i];
    seen[j] = 1;
  }
  for (int j = 0; j < S; ++j) {
    if (mx[j] > s->best_fitness[j]) { s->best_fitness[j] = mx[j]; s->stagnation[j] = 0; }
    else s->stagnation[j] += 1;
  }
  /* protection rank: max fitness desc, ties lower index */
  int* prot = (int*)calloc((size_t)S, sizeof(int));
  for (int j = 0; j < S; ++j) {
    int better = 0;
    for (int q = 0; q < S; ++q)
      if (mx[q] > mx[j] || (mx[q] == mx[j] && q < j)) ++better;
    if (better < cfg->species_elitism) prot[j] = 1;
  }
  int survivors = 0;
  for (int j = 0; j < S; ++j)
    if (prot[j] || s->stagnation[j] <= cfg->max_stagnation) ++survivors;
  if (survivors == 0) {
    int b = 0;
    for (int j = 1; j < S; ++j) if (mx[j] > mx[b]) b = j;
    prot[b] = 1;
  }
  int* remap = (int*)malloc(sizeof(int) * (size_t)S);
  int k = 0;
  for (int j = 0; j < S; ++j) {
    if (!prot[j] && s->stagnation[j] > cfg->max_stagnation) { remap[j] = -1; continue; }
    remap[j] = k++;
  }
  for (int j = 0; j < S; ++j) {  /* remap[j] <= j: forward compaction is safe */
    const int t = remap[j];
    if (t < 0 || t == j) continue;
    s->id[t] = s->id[j];
    s->best_fitness[t] = s->best_fitness[j];
    s->stagnation[t] = s->stagnation[j];
    s->size[t] = s->size[j];
    s->spawn[t] = s->spawn[j];
    memmove(s->rep_nodes + (size_t)t * s->nsz, s->rep_nodes + (size_t)j * s->nsz, sizeof(double) * s->nsz);
    memmove(s->rep_conns + (size_t)t * s->csz, s->rep_conns + (size_t)j * s->csz, sizeof(double) * s->csz);
  }
  s->count = k;
  for (int i = 0; i < P; ++i) if (species_of[i] >= 0) species_of[i] = remap[species_of[i]];
  free(remap);
  free(prot);
  free(mx);
  free(seen);
}

typedef struct { double f; int i; } fi_t;
static int fi_asc(const void* a, const void* b) {
  const fi_t* x = (const fi_t*)a; const fi_t* y = (const fi_t*)b;
  if (x->f != y->f) return x->f < y->f ? -1 : 1;
  return (x->i > y->i) - (x->i < y->i);
}
static int fi_desc(const void* a, const void* b) {
  const fi_t* x = (const fi_t*)a; const fi_t* y = (const fi_t*)b;
  if (x->f != y->f) return x->f > y->f ? -1 : 1;
  return (x->i > y->i) - (x->i < y->i);
}

void fo_compute_spawn(const fo_neat_cfg* cfg, const double* fitness,
                      const int* species_of, fo_species* s) {
  const int P = cfg->pop_size;
  const int S = s->count;
  /* mid-rank of fitness (ties share the mean of their positions, SPEC.md:
   * 374-382 "population ranks mapped to [0,1]"; the symmetric tie rule keeps
   * the SPEC example "identical fitness distributions -> equal split"):
   * 2 r_i = lo + hi - 1 for the tie group [lo, hi) of the ascending order.
   * The species mean of r_i/(P-1) is formed from the EXACT integer sum of
   * 2 r_i, so it does not depend on summation order:
   * af_j = double(sum 2 r_i) / ((2 (P-1)) * n_j). */
  fi_t* ord = (fi_t*)malloc(sizeof(fi_t) * (size_t)P);
  long long* rk = (long long*)malloc(sizeof(long long) * (size_t)P);
  for (int i = 0; i < P; ++i) { ord[i].f = fitness[i]; ord[i].i = i; }
  qsort(ord, (size_t)P, sizeof(fi_t), fi_asc);
  for (int lo = 0; lo < P;) {
    int hi = lo + 1;
    while (hi < P && ord[hi].f == ord[lo].f) ++hi;
    for (int r = lo; r < hi; ++r) rk[ord[r].i] = (long long)lo + (long long)hi - 1;
    lo = hi;
  }
  long long* rsum = (long long*)calloc((size_t)S, sizeof(long long));
  double* af = (double*)calloc((size_t)S, sizeof(double));
  int* cnt = (int*)calloc((size_t)S, sizeof(int));
  for (int i = 0; i < P; ++i) {
    const int j = species_of[i];
    if (j < 0) continue;
    rsum[j] += rk[i];
    cnt[j]++;
  }
  double total = 0.0;
  for (int j = 0; j < S; ++j) {
    af[j] = (double)rsum[j] / ((2.0 * (double)(P - 1)) * (double)cnt[j]);
    total += af[j];
  }
  double* nw = (double*)malloc(sizeof(double) * (size_t)S);
  double sum_new = 0.0;
  for (int j = 0; j < S; ++j) {
    const double target = total > 0.0 ? (af[j] / total) * (double)P : (double)P / (double)S;
    const double old = (double)cnt[j];
    const double md = round(cfg->spawn_number_change_rate * old);
    double v = target;
    if (v < old - md) v = old - md;
    if (v > old + md) v = old + md;
    nw[j] = v;
    sum_new += v;
  }
  int assigned = 0;
  double* frac = (double*)malloc(sizeof(double) * (size_t)S);
  for (int j = 0; j < S; ++j) {
    const double sc = sum_new > 0.0 ? (nw[j] * (double)P) / sum_new : (double)P / (double)S;
    const double fl = floor(sc);
    s->spawn[j] = (int)fl;
    frac[j] = sc - fl;
    assigned += s->spawn[j];
  }
  int rem = P - assigned;
  while (rem > 0) {
    int b = -1;
    for (int j = 0; j < S; ++j) if (frac[j] >= 0.0 && (b < 0 || frac[j] > frac[b])) b = j;
    if (b < 0) { for (int j = 0; j < S && rem > 0; ++j, --rem) s->spawn[j]++; break; }
    s->spawn[b]++;
    frac[b] = -1.0;
    --rem;
  }
  int tot = 0;
  for (int j = 0; j < S; ++j) {
    if (s->spawn[j] < cfg->genome_elitism) s->spawn[j] = cfg->genome_elitism;
    tot += s->spawn[j];
  }
  while (tot > P) {
    int b = -1;
    for (int j = 0; j < S; ++j)
      if (s->spawn[j] > cfg->genome_elitism && (b < 0 || s->spawn[j] >= s->spawn[b])) b = j;
    if (b < 0) break;
    s->spawn[b]--;
    --tot;
  }
  free(ord); free(rk); free(rsum); free(af); free(cnt); free(nw); free(frac);
}

int fo_reproduce(const fo_shape* sh, const fo_schema* sc, const fo_neat_cfg* cfg,
                 const double* pop_nodes, const double* pop_conns,
                 const double* fitness, const int* species_of,
                 const fo_species* s, uint64_t seed, int generation,
                 fo_innov* innov, double* next_nodes, double* next_conns,
                 int* parent_a, int* parent_b) {
  const int P = cfg->pop_size;
  const fo_key gk = fo_key_split(fo_key_split(fo_key_seed(seed), 1), (uint64_t)generation);
  fi_t* mem = (fi_t*)malloc(sizeof(fi_t) * (size_t)P);
  int slot = 0;
  int status = 0;
  for (int j = 0; j < s->count && !status; ++j) {
    int m = 0;
    for (int i = 0; i < P; ++i) if (species_of[i] == j) { mem[m].f = fitness[i]; mem[m].i = i; ++m; }
    qsort(mem, (size_t)m, sizeof(fi_t), fi_desc);
    int n_elite = cfg->genome_elitism;
    if (n_elite > s->spawn[j]) n_elite = s->spawn[j];
    if (n_elite > m) n_elite = m;
    int pool = (int)ceil(cfg->survival_threshold * (double)m);
    if (pool < 1) pool = 1;
    if (pool > m) pool = m;
    for (int k = 0; k < s->spawn[j] && slot < P; ++k, ++slot) {
      double* cn = next_nodes + (size_t)slot * NSZ(sh);
      double* cc = next_conns + (size_t)slot * CSZ(sh);
      if (k < n_elite) {
        const int e = mem[k].i;
        memcpy(cn, pop_nodes + (size_t)e * NSZ(sh), sizeof(double) * NSZ(sh));
        memcpy(cc, pop_conns + (size_t)e * CSZ(sh), sizeof(double) * CSZ(sh));
        parent_a[slot] = e;
        parent_b[slot] = -1;
        continue;
      }
      const fo_key ck = fo_key_split(gk, (uint64_t)slot);
      fo_stream sel;
      fo_stream_init(&sel, fo_key_split(ck, 0));
      const int a = mem[(int)fo_below(&sel, (uint64_t)pool)].i;
      const int b = mem[(int)fo_below(&sel, (uint64_t)pool)].i;
      int fit = a, oth = b;
      if (!(fitness[a] > fitness[b] || (fitness[a] == fitness[b] && a <= b))) { fit = b; oth = a; }
      parent_a[slot] = fit;
      parent_b[slot] = oth;
      fo_crossover(sh, pop_nodes + (size_t)fit * NSZ(sh), pop_conns + (size_t)fit * CSZ(sh),
                   pop_nodes + (size_t)oth * NSZ(sh), pop_conns + (size_t)oth * CSZ(sh),
                   fo_key_split(ck, 1), cn, cc);
      status = fo_mutate(sh, sc, cn, cc, fo_key_split(ck, 2), &cfg->mutation, innov);
      if (status) break;
    }
  }
  free(mem);
  return status;
}
