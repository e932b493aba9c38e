// flatneat/gpu.hpp -- B200 drop-in for the reference flatneat C++ API.
//
// Header-only C++20 wrapper over the C ABI (include/flatneat_b200.h) that
// speaks the reference's own types: include it NEXT TO the reference
// headers (proj/include/flatneat/*.hpp) and replace
//     transform + batch_forward   (network.hpp:122, 294)
//     distance                    (ops.hpp:415)
//     crossover                   (ops.hpp:382)
//     mutate with InnovationTable (ops.hpp:363, 145)
// by the flatneat::gpu:: calls below.  Errors come back as flatneat::Error
// with the reference's Errc and what() text (errors.hpp:59-73); link with
// paper_2504_08339_b200/libflatneat_b200.so.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "flatneat/errors.hpp"
#include "flatneat/genome.hpp"
#include "flatneat/network.hpp"
#include "flatneat/ops.hpp"
#include "flatneat/rng.hpp"
#include "flatneat_b200.h"

namespace flatneat::gpu {

namespace detail {

inline int builtin_activation(const std::string& n) {
  if (n == "identity") return FNB_ACT_IDENTITY;
  if (n == "tanh") return FNB_ACT_TANH;
  if (n == "sigmoid") return FNB_ACT_SIGMOID;
  if (n == "relu") return FNB_ACT_RELU;
  if (n == "sin") return FNB_ACT_SIN;
  raise(Errc::unknown_function, "activation '" + n + "' is not built in");
}
inline int builtin_aggregation(const std::string& n) {
  if (n == "sum") return FNB_AGG_SUM;
  if (n == "product") return FNB_AGG_PRODUCT;
  if (n == "max") return FNB_AGG_MAX;
  if (n == "mean") return FNB_AGG_MEAN;
  raise(Errc::unknown_function, "aggregation '" + n + "' is not built in");
}
inline fnb_attr_mutation attr(const AttrMutation& a) {
  return fnb_attr_mutation{a.init_mean, a.init_std, a.mutate_power, a.mutate_rate, a.replace_rate};
}
inline void copy_key(const RngKey& k, uint32_t* out) {
  for (int i = 0; i < 4; ++i) out[i] = k.words()[std::size_t(i)];
}

}  // namespace detail

// One device context for a fixed (limits, inputs, outputs, schema).
class Context {
 public:
  Context(GenomeLimits limits, std::vector<int> input_keys, std::vector<int> output_keys,
          const AttributeSchema& schema, int device = 0)
      : limits_(limits), in_(std::move(input_keys)), out_(std::move(output_keys)) {
    schema.check();
    fnb_schema sc{};
    sc.n_act = int(schema.activations.size());
    sc.n_agg = int(schema.aggregations.size());
    for (int i = 0; i < sc.n_act && i < 8; ++i) sc.act[i] = detail::builtin_activation(schema.activations[std::size_t(i)]);
    for (int i = 0; i < sc.n_agg && i < 8; ++i) sc.agg[i] = detail::builtin_aggregation(schema.aggregations[std::size_t(i)]);
    sc.default_act = schema.default_activation;
    sc.default_agg = schema.default_aggregation;
    const fnb_shape sh{limits.max_nodes, limits.max_conns, int(in_.size()), int(out_.size()), in_.data(),
                       out_.data()};
    if (const int st = fnb_ctx_create(&sh, &sc, device, &ctx_))
      throw Error(Errc(st - 1), "fnb_ctx_create failed");
  }
  ~Context() { fnb_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  // transform() of every genome (network.hpp:122): int32 orders, -1 padded
  std::vector<std::int32_t> transform_orders(const PopulationTensors& pop) {
    check_pop(pop);
    std::vector<std::int32_t> order(std::size_t(pop.pop_size) * std::size_t(limits_.max_nodes));
    check(fnb_transform(ctx_, pop.pop_nodes.data(), pop.pop_conns.data(), pop.pop_size, order.data(), nullptr));
    return order;
  }

  // transform + batch_forward (network.hpp:294-330); FP32 on the device
  BatchResult batch_forward(const PopulationTensors& pop, std::span<const double> inputs, int batch) {
    check_pop(pop);
    if (int(inputs.size()) != batch * int(in_.size()))
      raise(Errc::shape_mismatch, "input matrix is not batch x num_inputs");
    BatchResult r;
    r.pop_size = pop.pop_size;
    r.batch = batch;
    r.outputs = int(out_.size());
    r.values.resize(std::size_t(pop.pop_size) * std::size_t(batch) * out_.size());
    check(fnb_batch_forward(ctx_, pop.pop_nodes.data(), pop.pop_conns.data(), pop.pop_size, inputs.data(), batch,
                            r.values.data()));
    return r;
  }

  // transform + forward + fused fitness: fitness_kind is
  // FNB_FIT_NEG_MSE (func-fit) or FNB_FIT_OFFSET_SSE (xor, `offset` - SSE)
  std::vector<double> evaluate(const PopulationTensors& pop, std::span<const double> inputs,
                               std::span<const double> targets, int batch, int fitness_kind = FNB_FIT_NEG_MSE,
                               double offset = 0.0) {
    check_pop(pop);
    if (int(inputs.size()) != batch * int(in_.size()) || int(targets.size()) != batch * int(out_.size()))
      raise(Errc::shape_mismatch, "input / target matrix is not batch x num_inputs / num_outputs");
    std::vector<double> fit(std::size_t(pop.pop_size));
    check(fnb_evaluate(ctx_, pop.pop_nodes.data(), pop.pop_conns.data(), pop.pop_size, inputs.data(),
                       targets.data(), batch, fitness_kind, offset, fit.data()));
    return fit;
  }

  // distance(genome_p, rep_s) (ops.hpp:415) for a population x representatives
  std::vector<double> distance(const PopulationTensors& pop, const PopulationTensors& reps,
                               const DistanceConfig& cfg = {}) {
    check_pop(pop);
    check_pop(reps);
    std::vector<double> out(std::size_t(pop.pop_size) * std::size_t(reps.pop_size));
    const fnb_distance_config dc{cfg.compatibility_disjoint, cfg.compatibility_homologous};
    check(fnb_distance(ctx_, pop.pop_nodes.data(), pop.pop_conns.data(), pop.pop_size, reps.pop_nodes.data(),
                       reps.pop_conns.data(), reps.pop_size, &dc, out.data()));
    return out;
  }

  // crossover(fit[i], other[i], keys[i]) (ops.hpp:382) pairwise
  PopulationTensors crossover(const PopulationTensors& fit, const PopulationTensors& other,
                              std::span<const RngKey> keys) {
    check_pop(fit);
    check_pop(other);
    if (other.pop_size != fit.pop_size || int(keys.size()) != fit.pop_size)
      raise(Errc::shape_mismatch, "crossover needs one other parent and one key per fit parent");
    std::vector<std::uint32_t> k(keys.size() * 4);
    for (std::size_t i = 0; i < keys.size(); ++i) detail::copy_key(keys[i], k.data() + 4 * i);
    PopulationTensors child = fit;
    check(fnb_crossover(ctx_, fit.pop_nodes.data(), fit.pop_conns.data(), other.pop_nodes.data(),
                        other.pop_conns.data(), fit.pop_size, k.data(), child.pop_nodes.data(),
                        child.pop_conns.data()));
    return child;
  }

  // mutate(genome_p, keys[p], cfg, schema, table) for p in slot order with
  // the caller's InnovationTable (ops.hpp:169-175, 363): the table's
  // get_or_assign is called once per splitting slot, in slot order, so its
  // memo and counter end exactly as the sequential loop leaves them --
  // including entries it already held from earlier calls this generation.
  // On error, genomes before the failing slot are mutated and the rest untouched.
  void mutate(PopulationTensors& pop, std::span<const RngKey> keys, const MutationConfig& cfg,
              InnovationTable& table) {
    check_pop(pop);
    if (int(keys.size()) != pop.pop_size) raise(Errc::shape_mismatch, "mutate needs one key per genome");
    std::vector<std::uint32_t> k(keys.size() * 4);
    for (std::size_t i = 0; i < keys.size(); ++i) detail::copy_key(keys[i], k.data() + 4 * i);
    const fnb_mutation_config mc{cfg.node_add, cfg.node_delete, cfg.conn_add, cfg.conn_delete,
                                 detail::attr(cfg.bias), detail::attr(cfg.response), detail::attr(cfg.weight),
                                 cfg.activation_replace_rate, cfg.aggregation_replace_rate};
    auto thunk = [](void* user, int in_key, int out_key) -> int {
      return static_cast<InnovationTable*>(user)->get_or_assign(in_key, out_key);
    };
    check(fnb_mutate_table(ctx_, pop.pop_nodes.data(), pop.pop_conns.data(), pop.pop_size, k.data(), &mc, thunk,
                           &table, nullptr));
  }

  fnb_ctx* handle() { return ctx_; }
  // a nonzero ABI status as flatneat::Error with the reference's Errc and text
  void rethrow(int st) { check(st); }

 private:
  // the flat arrays must hold pop_size genomes of this context's limits
  // (PopulationTensors layout, genome.hpp:315-338)
  void check_pop(const PopulationTensors& p) const {
    if (p.limits.max_nodes != limits_.max_nodes || p.limits.max_conns != limits_.max_conns || p.pop_size < 0 ||
        p.pop_nodes.size() != std::size_t(p.pop_size) * std::size_t(limits_.max_nodes) * kNodeCols ||
        p.pop_conns.size() != std::size_t(p.pop_size) * std::size_t(limits_.max_conns) * kConnCols)
      raise(Errc::shape_mismatch, "population tensors do not match the context's limits");
  }

  void check(int st) {
    if (!st) return;
    const std::string what = fnb_last_error(ctx_);
    const auto colon = what.find(": ");
    throw Error(Errc(st - 1), colon == std::string::npos ? what : what.substr(colon + 2));
  }

  GenomeLimits limits_;
  std::vector<int> in_, out_;
  fnb_ctx* ctx_ = nullptr;
};

// SPEC's evolution module on the device: the population,
// species table and innovation counter stay in HBM.  NeatConfig is SPEC-only
// (the reference has no type for it), so the C struct is used as is.
struct RunStats {
  int generation = 0;
  double best = 0, mean = 0, std = 0;
  int best_index = -1;
  std::vector<int> species_sizes;  // one entry per species
  double elapsed_ms = 0;
};

struct EvolveResult {
  GenomeTensors best;      // pop[argmax(fit)] of the last evaluated generation
  double fitness = 0;
  std::vector<RunStats> stats;
};

// Checkpoint of everything a generation step reads (fnb_evolver_get_state).
struct EvolverState {
  fnb_run_state state{};
  PopulationTensors representatives;
  PopulationTensors population;
};

class Evolver {
 public:
  Evolver(Context& ctx, const fnb_neat_config& cfg, std::uint64_t seed, GenomeLimits limits,
          std::vector<int> input_keys, std::vector<int> output_keys)
      : ctx_(ctx), cfg_(cfg), limits_(limits), in_(std::move(input_keys)), out_(std::move(output_keys)) {
    if (const int st = fnb_evolver_create(ctx_.handle(), &cfg_, seed, &ev_)) ctx_.rethrow(st);
  }
  ~Evolver() { fnb_evolver_destroy(ev_); }
  Evolver(const Evolver&) = delete;
  Evolver& operator=(const Evolver&) = delete;

  void init_population() { ctx_.rethrow(fnb_evolver_init_population(ev_)); }

  PopulationTensors population() {
    PopulationTensors p = empty(cfg_.pop_size);
    ctx_.rethrow(fnb_evolver_get_population(ev_, p.pop_nodes.data(), p.pop_conns.data()));
    return p;
  }
  // loads a population; the innovation counter moves above its largest key
  void set_population(const PopulationTensors& p) {
    if (p.pop_size != cfg_.pop_size || p.limits.max_nodes != limits_.max_nodes ||
        p.limits.max_conns != limits_.max_conns)
      raise(Errc::shape_mismatch, "population does not match the evolver");
    ctx_.rethrow(fnb_evolver_set_population(ev_, p.pop_nodes.data(), p.pop_conns.data()));
    int top = 0;
    for (std::size_t i = 0; i < p.pop_nodes.size(); i += kNodeCols)
      if (!std::isnan(p.pop_nodes[i])) top = std::max(top, int(p.pop_nodes[i]) + 1);
    int gen = 0, nk = 0;
    ctx_.rethrow(fnb_evolver_state(ev_, &gen, &nk));
    ctx_.rethrow(fnb_evolver_set_next_key(ev_, std::max(top, nk)));
  }

  // evolve(problem, cfg, key) on a func-fit / xor dataset
  EvolveResult evolve(std::span<const double> inputs, std::span<const double> targets, int batch,
                      double fitness_target, int generation_limit, int fitness_kind = FNB_FIT_NEG_MSE,
                      double offset = 0.0, const std::function<bool(const RunStats&)>& on_generation = {}) {
    if (int(inputs.size()) != batch * int(in_.size()) || int(targets.size()) != batch * int(out_.size()))
      raise(Errc::shape_mismatch, "input / target matrix is not batch x num_inputs / num_outputs");
    struct Ctx {
      std::vector<RunStats>* out;
      const std::function<bool(const RunStats&)>* cb;
    };
    EvolveResult r{GenomeTensors(limits_, in_, out_), 0.0, {}};
    Ctx c{&r.stats, &on_generation};
    auto thunk = [](void* user, const fnb_run_stats* s) -> int {
      auto* c = static_cast<Ctx*>(user);
      RunStats rs;
      rs.generation = s->generation;
      rs.best = s->best;
      rs.mean = s->mean;
      rs.std = s->std;
      rs.best_index = s->best_index;
      rs.species_sizes.assign(s->species_size, s->species_size + s->species_count);
      rs.elapsed_ms = s->elapsed_ms;
      c->out->push_back(rs);
      return (*c->cb && (*c->cb)(c->out->back())) ? 1 : 0;
    };
    int gens = 0;
    ctx_.rethrow(fnb_evolve(ev_, inputs.data(), targets.data(), batch, fitness_kind, offset, fitness_target,
                            generation_limit, thunk, &c, r.best.nodes.data(), r.best.conns.data(), &r.fitness, &gens));
    return r;
  }

  EvolverState save() {
    EvolverState s;
    s.representatives = empty(32);
    ctx_.rethrow(fnb_evolver_get_state(ev_, &s.state, s.representatives.pop_nodes.data(),
                                       s.representatives.pop_conns.data()));
    s.representatives.pop_size = s.state.species_count;
    s.representatives.pop_nodes.resize(std::size_t(s.state.species_count) * limits_.max_nodes * kNodeCols);
    s.representatives.pop_conns.resize(std::size_t(s.state.species_count) * limits_.max_conns * kConnCols);
    s.population = population();
    return s;
  }
  void restore(const EvolverState& s) {
    ctx_.rethrow(fnb_evolver_set_population(ev_, s.population.pop_nodes.data(), s.population.pop_conns.data()));
    ctx_.rethrow(fnb_evolver_set_state(ev_, &s.state, s.representatives.pop_nodes.data(),
                                       s.representatives.pop_conns.data()));
  }

  fnb_evolver* handle() { return ev_; }

 private:
  PopulationTensors empty(int n) const {
    PopulationTensors p;
    p.pop_size = n;
    p.limits = limits_;
    p.input_keys = in_;
    p.output_keys = out_;
    p.pop_nodes.assign(std::size_t(n) * limits_.max_nodes * kNodeCols, kNaN);
    p.pop_conns.assign(std::size_t(n) * limits_.max_conns * kConnCols, kNaN);
    return p;
  }

  Context& ctx_;
  fnb_neat_config cfg_;
  GenomeLimits limits_;
  std::vector<int> in_, out_;
  fnb_evolver* ev_ = nullptr;
};

}  // namespace flatneat::gpu
