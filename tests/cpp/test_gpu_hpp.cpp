// C++ drop-in check -- TEST ONLY.  Uses the reference's own types and
// functions (the unmodified /root/reference headers, compiled in) next to
// flatneat::gpu (include/flatneat/gpu.hpp) and compares:
//   batch_forward  within 1e-5 rel + 1e-5 abs (FP32 device, FP64 reference)
//   distance, crossover, mutate (+ InnovationTable counter)  bit for bit
// Prints "gpu.hpp parity ok" and exits 0 on success.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "flatneat/genome.hpp"
#include "flatneat/gpu.hpp"
#include "flatneat/network.hpp"
#include "flatneat/ops.hpp"
#include "support/generators.hpp"

using namespace flatneat;

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  if (a.size() != b.size()) return false;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const bool na = std::isnan(a[i]), nb = std::isnan(b[i]);
    if (na != nb || (!na && std::memcmp(&a[i], &b[i], 8) != 0)) return false;
  }
  return true;
}

int main() {
  AttributeSchema s;
  s.activations = {"tanh", "sigmoid", "identity", "relu", "sin"};
  s.aggregations = {"sum", "product", "max", "mean"};
  const GenomeLimits lim{24, 80};
  RngStream stream{RngKey(1312)};
  std::vector<GenomeTensors> gs;
  for (int i = 0; i < 96; ++i) gs.push_back(testgen::random_acyclic_genome(stream, s).pad(lim));
  const PopulationTensors pop = concat_population(gs);
  gpu::Context ctx(lim, pop.input_keys, pop.output_keys, s);
  int fails = 0;

  // forward
  std::vector<double> X;
  for (int i = 0; i < 64 * 3; ++i) X.push_back(stream.uniform(-2, 2));
  std::vector<TransformedNetwork> nets;
  for (const auto& g : gs) nets.push_back(transform(g, s));
  const BatchResult want = batch_forward(nets, X, 64);
  const BatchResult got = ctx.batch_forward(pop, X, 64);
  for (std::size_t i = 0; i < want.values.size(); ++i)
    if (std::fabs(got.values[i] - want.values[i]) > 1e-5 + 1e-5 * std::fabs(want.values[i])) { ++fails; break; }

  // distance
  std::vector<GenomeTensors> rv(gs.begin(), gs.begin() + 5);
  const PopulationTensors reps = concat_population(rv);
  const auto d = ctx.distance(pop, reps);
  for (int p = 0; p < pop.pop_size; ++p)
    for (int r = 0; r < reps.pop_size; ++r) {
      const double w = distance(gs[std::size_t(p)], rv[std::size_t(r)], DistanceConfig{});
      if (std::memcmp(&w, &d[std::size_t(p) * reps.pop_size + r], 8) != 0) ++fails;
    }

  // crossover
  std::vector<RngKey> keys;
  for (int i = 0; i < pop.pop_size; ++i) keys.push_back(RngKey(9).split(std::uint64_t(i)));
  std::vector<GenomeTensors> other(gs.rbegin(), gs.rend());
  const PopulationTensors opop = concat_population(other);
  const PopulationTensors child = ctx.crossover(pop, opop, keys);
  for (int i = 0; i < pop.pop_size; ++i) {
    const auto c = crossover(gs[std::size_t(i)], other[std::size_t(i)], keys[std::size_t(i)]);
    if (!(child.slice(i) == c)) ++fails;
  }

  // mutate with one table, slot order
  MutationConfig mc;
  mc.node_delete = 0.1;
  mc.conn_delete = 0.1;
  InnovationTable tref(1000), tgpu(1000);
  PopulationTensors mp = pop;
  ctx.mutate(mp, keys, mc, tgpu);
  for (int i = 0; i < pop.pop_size; ++i) {
    const auto m = mutate(gs[std::size_t(i)], keys[std::size_t(i)], mc, s, tref);
    if (!(mp.slice(i) == m)) ++fails;
  }
  if (tref.next_key() != tgpu.next_key()) ++fails;

  std::printf(fails ? "gpu.hpp parity FAILED (%d)\n" : "gpu.hpp parity ok\n", fails);
  return fails ? 1 : 0;
}
