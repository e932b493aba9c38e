// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference headers
// (/root/reference/proj/include/flatneat/*.hpp and
// /root/reference/proj/tests/support/generators.hpp), compiled by
// oracle/Makefile into oracle/_ref/libflatneat_ref.so.  No reference source
// is copied: the headers are #included from where they lie.  The library is
// the strongest oracle we have: tests use it to pin the C restatement
// (oracle/flatneat_oracle.c), to dump golden vectors, and bench.py's
// --impl reference / cpu_baseline leg times the reference's own
// batch_forward on the host cores through it.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "flatneat/errors.hpp"
#include "flatneat/functions.hpp"
#include "flatneat/genome.hpp"
#include "flatneat/network.hpp"
#include "flatneat/ops.hpp"
#include "flatneat/parallel.hpp"
#include "flatneat/rng.hpp"
#include "support/generators.hpp"

#include "flatneat_oracle.h"  // POD shapes/configs only; no oracle code is called

using namespace flatneat;

namespace {

const char* kActNames[] = {"identity", "tanh", "sigmoid", "relu", "sin"};
const char* kAggNames[] = {"sum", "product", "max", "mean"};

AttributeSchema to_schema(const fo_schema* sc) {
  AttributeSchema s;
  s.activations.clear();
  s.aggregations.clear();
  for (int i = 0; i < sc->n_act; ++i) s.activations.push_back(kActNames[sc->act[i]]);
  for (int i = 0; i < sc->n_agg; ++i) s.aggregations.push_back(kAggNames[sc->agg[i]]);
  s.default_activation = sc->default_act;
  s.default_aggregation = sc->default_agg;
  return s;
}

GenomeTensors to_genome(const fo_shape* sh, const double* nodes, const double* conns) {
  GenomeTensors g(GenomeLimits{sh->max_nodes, sh->max_conns},
                  std::vector<int>(sh->input_keys, sh->input_keys + sh->num_inputs),
                  std::vector<int>(sh->output_keys, sh->output_keys + sh->num_outputs));
  std::memcpy(g.nodes.data(), nodes, sizeof(double) * g.nodes.size());
  std::memcpy(g.conns.data(), conns, sizeof(double) * g.conns.size());
  return g;
}

void from_genome(const GenomeTensors& g, double* nodes, double* conns) {
  std::memcpy(nodes, g.nodes.data(), sizeof(double) * g.nodes.size());
  std::memcpy(conns, g.conns.data(), sizeof(double) * g.conns.size());
}

RngKey to_key(const uint32_t w[4]) {
  static_assert(sizeof(RngKey) == 16, "RngKey layout");
  RngKey k;
  std::memcpy(static_cast<void*>(&k), w, 16);
  return k;
}

MutationConfig to_mut(const fo_mut_cfg* c) {
  MutationConfig m;
  m.node_add = c->node_add;
  m.node_delete = c->node_delete;
  m.conn_add = c->conn_add;
  m.conn_delete = c->conn_delete;
  auto cv = [](const fo_attr_mut& a) {
    return AttrMutation{a.init_mean, a.init_std, a.mutate_power, a.mutate_rate, a.replace_rate};
  };
  m.bias = cv(c->bias);
  m.response = cv(c->response);
  m.weight = cv(c->weight);
  m.activation_replace_rate = c->activation_replace_rate;
  m.aggregation_replace_rate = c->aggregation_replace_rate;
  return m;
}

int report(const Error& e, char* msg, size_t n) {
  if (msg && n) {
    std::strncpy(msg, e.what(), n - 1);
    msg[n - 1] = 0;
  }
  return 1 + int(e.code());
}

}  // namespace

extern "C" {

void fr_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  auto b = detail::philox4x32_10({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = b.w[std::size_t(i)];
}

void fr_key_seed(uint64_t seed, uint32_t out[4]) {
  RngKey k(seed);
  for (int i = 0; i < 4; ++i) out[i] = k.words()[std::size_t(i)];
}

void fr_key_split(const uint32_t w[4], uint64_t index, uint32_t out[4]) {
  RngKey k = to_key(w).split(index);
  for (int i = 0; i < 4; ++i) out[i] = k.words()[std::size_t(i)];
}

// kind 0: next_u64 (out_u), 1: uniform, 2: normal(a, b), 3: below(n=a), 4: coin(p=a)
void fr_stream_draws(const uint32_t w[4], int kind, int n, double a, double b,
                     uint64_t* out_u, double* out_d) {
  RngStream s(to_key(w));
  for (int i = 0; i < n; ++i) {
    switch (kind) {
      case 0: out_u[i] = s.next_u64(); break;
      case 1: out_d[i] = s.uniform(); break;
      case 2: out_d[i] = s.normal(a, b); break;
      case 3: out_u[i] = s.below(uint64_t(a)); break;
      case 4: out_u[i] = s.coin(a) ? 1 : 0; break;
    }
  }
}

int fr_transform(const fo_shape* sh, const fo_schema* sc, const double* nodes,
                 const double* conns, int32_t* order, int* order_count,
                 double* expanded, int* input_rows, int* output_rows, char* msg,
                 size_t msg_n) {
  try {
    const auto t = transform(to_genome(sh, nodes, conns), to_schema(sc));
    for (int i = 0; i < sh->max_nodes; ++i) order[i] = t.order[std::size_t(i)];
    *order_count = t.order_count;
    if (expanded) std::memcpy(expanded, t.expanded.data(), sizeof(double) * t.expanded.size());
    for (int i = 0; i < sh->num_inputs; ++i) input_rows[i] = t.input_rows[std::size_t(i)];
    for (int i = 0; i < sh->num_outputs; ++i) output_rows[i] = t.output_rows[std::size_t(i)];
    return 0;
  } catch (const Error& e) {
    return report(e, msg, msg_n);
  }
}

// transform + batch_forward over a population (network.hpp:122, :294).
// status: lowest-index failure; nthreads<=1 runs inline.
int fr_batch_forward(const fo_shape* sh, const fo_schema* sc, int P,
                     const double* pop_nodes, const double* pop_conns,
                     const double* inputs, int batch, double* out, int nthreads,
                     int* bad_genome, char* msg, size_t msg_n) {
  const auto schema = to_schema(sc);
  const std::size_t ns = std::size_t(sh->max_nodes) * kNodeCols;
  const std::size_t cs = std::size_t(sh->max_conns) * kConnCols;
  std::vector<TransformedNetwork> nets(static_cast<std::size_t>(P));
  std::vector<int> status(static_cast<std::size_t>(P), 0);
  std::vector<std::string> msgs(static_cast<std::size_t>(P));
  auto body = [&](int lo, int hi) {
    for (int p = lo; p < hi; ++p) {
      try {
        nets[std::size_t(p)] = transform(
            to_genome(sh, pop_nodes + std::size_t(p) * ns, pop_conns + std::size_t(p) * cs), schema);
      } catch (const Error& e) {
        status[std::size_t(p)] = 1 + int(e.code());
        msgs[std::size_t(p)] = e.what();
      }
    }
  };
  std::unique_ptr<ThreadPool> pool;
  if (nthreads > 1) pool = std::make_unique<ThreadPool>(nthreads);
  parallel_for(pool.get(), P, 16, body);
  for (int p = 0; p < P; ++p) {
    if (status[std::size_t(p)]) {
      if (bad_genome) *bad_genome = p;
      if (msg && msg_n) {
        std::strncpy(msg, msgs[std::size_t(p)].c_str(), msg_n - 1);
        msg[msg_n - 1] = 0;
      }
      return status[std::size_t(p)];
    }
  }
  try {
    const auto r = batch_forward(nets, std::span<const double>(inputs, std::size_t(batch) * std::size_t(sh->num_inputs)),
                                 batch, pool.get(), 16);
    if (out) std::memcpy(out, r.values.data(), sizeof(double) * r.values.size());
  } catch (const Error& e) {
    if (bad_genome) *bad_genome = -1;
    return report(e, msg, msg_n);
  }
  return 0;
}

double fr_distance(const fo_shape* sh, const double* n1, const double* c1,
                   const double* n2, const double* c2, const fo_dist_cfg* cfg) {
  return distance(to_genome(sh, n1, c1), to_genome(sh, n2, c2),
                  DistanceConfig{cfg->compatibility_disjoint, cfg->compatibility_homologous});
}

void fr_crossover(const fo_shape* sh, const double* fn, const double* fc, const double* on,
                  const double* oc, const uint32_t key[4], double* cn, double* cc) {
  const auto child = crossover(to_genome(sh, fn, fc), to_genome(sh, on, oc), to_key(key));
  from_genome(child, cn, cc);
}

// distance(genome_p, rep_s) for a population x S representatives with the
// reference's parallel_for over the population (parallel.hpp:74-110) --
// bench.py's CPU generation baseline.  out[P][S].
void fr_distance_matrix(const fo_shape* sh, int P, const double* pop_nodes, const double* pop_conns, int S,
                        const double* rep_nodes, const double* rep_conns, const fo_dist_cfg* cfg, int nthreads,
                        double* out) {
  const std::size_t ns = std::size_t(sh->max_nodes) * kNodeCols;
  const std::size_t cs = std::size_t(sh->max_conns) * kConnCols;
  const DistanceConfig dc{cfg->compatibility_disjoint, cfg->compatibility_homologous};
  std::vector<GenomeTensors> reps;
  for (int s = 0; s < S; ++s) reps.push_back(to_genome(sh, rep_nodes + std::size_t(s) * ns, rep_conns + std::size_t(s) * cs));
  std::unique_ptr<ThreadPool> pool;
  if (nthreads > 1) pool = std::make_unique<ThreadPool>(nthreads);
  parallel_for(pool.get(), P, 16, [&](int lo, int hi) {
    for (int p = lo; p < hi; ++p) {
      const auto g = to_genome(sh, pop_nodes + std::size_t(p) * ns, pop_conns + std::size_t(p) * cs);
      for (int s = 0; s < S; ++s) out[std::size_t(p) * S + s] = distance(g, reps[std::size_t(s)], dc);
    }
  });
}

// crossover(fit[c], other[c], keys[c]) for c < n, one thread (the per-slot
// loop of reproduce) -- bench.py's CPU generation baseline.
void fr_crossover_population(const fo_shape* sh, int n, const double* fit_nodes, const double* fit_conns,
                             const double* oth_nodes, const double* oth_conns, const uint32_t* keys,
                             double* child_nodes, double* child_conns) {
  const std::size_t ns = std::size_t(sh->max_nodes) * kNodeCols;
  const std::size_t cs = std::size_t(sh->max_conns) * kConnCols;
  for (int c = 0; c < n; ++c) {
    const auto child = crossover(to_genome(sh, fit_nodes + std::size_t(c) * ns, fit_conns + std::size_t(c) * cs),
                                 to_genome(sh, oth_nodes + std::size_t(c) * ns, oth_conns + std::size_t(c) * cs),
                                 to_key(keys + 4 * c));
    from_genome(child, child_nodes + std::size_t(c) * ns, child_conns + std::size_t(c) * cs);
  }
}

// Sequential mutate of P genomes in slot order with ONE InnovationTable, the
// population-level pattern of ops.hpp:169-175.  keys: P*4 words.  In place.
int fr_mutate_population(const fo_shape* sh, const fo_schema* sc, int P, double* pop_nodes,
                         double* pop_conns, const uint32_t* keys, const fo_mut_cfg* cfg,
                         int* next_key, int* bad_genome, char* msg, size_t msg_n) {
  const auto schema = to_schema(sc);
  const auto m = to_mut(cfg);
  InnovationTable table(*next_key);
  const std::size_t ns = std::size_t(sh->max_nodes) * kNodeCols;
  const std::size_t cs = std::size_t(sh->max_conns) * kConnCols;
  for (int p = 0; p < P; ++p) {
    try {
      const auto g = to_genome(sh, pop_nodes + std::size_t(p) * ns, pop_conns + std::size_t(p) * cs);
      const auto out = mutate(g, to_key(keys + 4 * p), m, schema, table);
      from_genome(out, pop_nodes + std::size_t(p) * ns, pop_conns + std::size_t(p) * cs);
    } catch (const Error& e) {
      if (bad_genome) *bad_genome = p;
      *next_key = table.next_key();
      return report(e, msg, msg_n);
    }
  }
  *next_key = table.next_key();
  return 0;
}

// testgen::random_acyclic_genome (generators.hpp:37-84) drawn from a stream
// positioned after `skip` genomes of the same spec (so callers can slice).
int fr_random_genomes(uint64_t seed, const fo_schema* sc, const fo_genspec* spec, int count,
                      int max_nodes, int max_conns, double* nodes, double* conns) {
  const auto schema = to_schema(sc);
  RngStream stream{RngKey(seed)};
  testgen::GenomeSpec gs{spec->num_inputs, spec->num_outputs, spec->max_hidden, spec->conn_prob,
                         spec->disabled_prob};
  const std::size_t ns = std::size_t(max_nodes) * kNodeCols;
  const std::size_t cs = std::size_t(max_conns) * kConnCols;
  for (int i = 0; i < count; ++i) {
    try {
      const auto g = testgen::random_acyclic_genome(stream, schema, gs).pad(GenomeLimits{max_nodes, max_conns});
      from_genome(g, nodes + std::size_t(i) * ns, conns + std::size_t(i) * cs);
    } catch (const Error& e) {
      return 1 + int(e.code());
    }
  }
  return 0;
}

// explain_invalid (genome.hpp:364-417); returns 1 if invalid.
int fr_explain_invalid(const fo_shape* sh, const fo_schema* sc, const double* nodes,
                       const double* conns, char* buf, size_t n) {
  const auto s = explain_invalid(to_genome(sh, nodes, conns), to_schema(sc));
  if (n) {
    std::strncpy(buf, s.c_str(), n - 1);
    buf[n - 1] = 0;
  }
  return s.empty() ? 0 : 1;
}

int fr_hardware_threads() { return int(std::thread::hardware_concurrency()); }

}  // extern "C"
