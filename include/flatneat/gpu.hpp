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

#include <cstring>
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

}  // namespace flatneat::gpu
