// C++ drop-in check -- TEST ONLY.  Uses the reference's own types and
// functions (the unmodified /root/reference headers, compiled in) next to
// flatneat::gpu (include/flatneat/gpu.hpp) and compares:
//   batch_forward  within 1e-5 rel + 1e-5 abs (FP32 device, FP64 reference)
//   distance, crossover, mutate (+ InnovationTable counter)  bit for bit
// Prints "gpu.hpp parity ok" and exits 0 on success.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
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

  // a pre-seeded table, and reference / GPU mutate calls mixed within one
  // generation: the memo must carry across them (ops.hpp:145-175)
  {
    InnovationTable ra(2000), ga(2000);
    for (int i = 0; i < pop.pop_size; i += 3) {  // seed the splits some slots will plan
      const NodeSplitPlan pl = plan_node_split(gs[std::size_t(i)], keys[std::size_t(i)], mc);
      if (pl.split) { ra.get_or_assign(pl.in_key, pl.out_key); ga.get_or_assign(pl.in_key, pl.out_key); }
    }
    const int half = pop.pop_size / 2;
    std::vector<GenomeTensors> want_m;
    for (int i = 0; i < pop.pop_size; ++i) want_m.push_back(mutate(gs[std::size_t(i)], keys[std::size_t(i)], mc, s, ra));
    // slots [0, half) on the reference, [half, P) on the GPU, one table
    std::vector<GenomeTensors> first;
    for (int i = 0; i < half; ++i) first.push_back(mutate(gs[std::size_t(i)], keys[std::size_t(i)], mc, s, ga));
    std::vector<GenomeTensors> second(gs.begin() + half, gs.end());
    PopulationTensors sp = concat_population(second);
    ctx.mutate(sp, std::span<const RngKey>(keys).subspan(std::size_t(half)), mc, ga);
    for (int i = 0; i < half; ++i)
      if (!(first[std::size_t(i)] == want_m[std::size_t(i)])) ++fails;
    for (int i = half; i < pop.pop_size; ++i)
      if (!(sp.slice(i - half) == want_m[std::size_t(i)])) { std::printf("mixed slot %d differs\n", i); ++fails; }
    // the memo: every pair the reference table knows maps to the same key
    for (int i = 0; i < pop.pop_size; ++i) {
      const NodeSplitPlan pl = plan_node_split(gs[std::size_t(i)], keys[std::size_t(i)], mc);
      if (pl.split && ra.get_or_assign(pl.in_key, pl.out_key) != ga.get_or_assign(pl.in_key, pl.out_key)) ++fails;
    }
    if (ra.next_key() != ga.next_key()) ++fails;
  }

  // duplicate_key: a table whose counter runs into existing node keys throws
  // at the first colliding slot; earlier genomes are mutated, later ones not
  {
    MutationConfig m2;
    m2.node_add = 1.0;
    InnovationTable ra(0), ga(0);
    int ref_bad = -1;
    std::string ref_what;
    std::vector<GenomeTensors> want_m;
    for (int i = 0; i < pop.pop_size; ++i) {
      try {
        want_m.push_back(mutate(gs[std::size_t(i)], keys[std::size_t(i)], m2, s, ra));
      } catch (const Error& e) {
        ref_bad = i;
        ref_what = e.what();
        break;
      }
    }
    PopulationTensors dp = pop;
    int gpu_bad = -1;
    std::string gpu_what;
    try {
      ctx.mutate(dp, keys, m2, ga);
    } catch (const Error& e) {
      gpu_bad = fnb_last_error_index(ctx.handle());
      gpu_what = e.what();
    }
    if (ref_bad < 0 || gpu_bad != ref_bad || gpu_what != ref_what || ra.next_key() != ga.next_key()) {
      std::printf("duplicate_key: ref slot %d '%s' next %d, gpu slot %d '%s' next %d\n", ref_bad, ref_what.c_str(),
                  ra.next_key(), gpu_bad, gpu_what.c_str(), ga.next_key());
      ++fails;
    }
    for (int i = 0; i < pop.pop_size; ++i) {
      const bool ok = i < ref_bad ? dp.slice(i) == want_m[std::size_t(i)] : dp.slice(i) == gs[std::size_t(i)];
      if (!ok) { std::printf("duplicate_key: genome %d\n", i); ++fails; break; }
    }
  }

  // span sizes and the empty dataset
  {
    bool threw = false;
    try {
      PopulationTensors q = pop;
      ctx.mutate(q, std::span<const RngKey>(keys).first(3), mc, tgpu);
    } catch (const Error& e) {
      threw = e.code() == Errc::shape_mismatch;
    }
    if (!threw) { std::printf("short key span accepted\n"); ++fails; }
    threw = false;
    try {
      PopulationTensors q = opop;
      q.pop_size = pop.pop_size + 1;
      (void)ctx.crossover(pop, q, keys);
    } catch (const Error& e) {
      threw = e.code() == Errc::shape_mismatch;
    }
    if (!threw) { std::printf("short other population accepted\n"); ++fails; }
    threw = false;
    try {
      (void)ctx.evaluate(pop, std::span<const double>(), std::span<const double>(), 0);
    } catch (const Error& e) {
      threw = e.code() == Errc::empty_dataset;
    }
    if (!threw) { std::printf("empty dataset accepted\n"); ++fails; }
  }

  // the evolver wrapper: evolve() with RunStats, save / restore continuing bit for bit
  {
    const GenomeLimits el{20, 60};
    gpu::Context ectx(el, {0, 1, 2}, {3}, s);
    fnb_neat_config nc{};
    nc.pop_size = 200;
    nc.max_species = 6;
    nc.compatibility_threshold = 0.8;
    nc.species_elitism = 2;
    nc.max_stagnation = 15;
    nc.genome_elitism = 2;
    nc.survival_threshold = 0.2;
    nc.spawn_number_change_rate = 0.5;
    nc.output_activation = 0;
    nc.mutation = fnb_mutation_config{0.3, 0.05, 0.5, 0.05, {0.0, 1.0, 0.5, 0.7, 0.1}, {1.0, 0.0, 0.0, 0.0, 0.0},
                                      {0.0, 1.0, 0.5, 0.8, 0.1}, 0.0, 0.0};
    nc.distance = fnb_distance_config{1.0, 0.5};
    std::vector<double> ex, ey;
    for (int b = 0; b < 32; ++b) {
      double t = 0;
      for (int i = 0; i < 3; ++i) { ex.push_back(stream.uniform(-1, 1)); t += ex.back(); }
      ey.push_back(std::tanh(t));
    }
    gpu::Evolver full(ectx, nc, 77, el, {0, 1, 2}, {3});
    full.init_population();
    const auto all = full.evolve(ex, ey, 32, std::numeric_limits<double>::infinity(), 12);
    gpu::Evolver part(ectx, nc, 77, el, {0, 1, 2}, {3});
    part.init_population();
    part.evolve(ex, ey, 32, std::numeric_limits<double>::infinity(), 6);
    const gpu::EvolverState st = part.save();
    gpu::Evolver resumed(ectx, nc, 1, el, {0, 1, 2}, {3});
    resumed.restore(st);
    const auto rest = resumed.evolve(ex, ey, 32, std::numeric_limits<double>::infinity(), 6);
    if (all.stats.size() != 12 || rest.stats.size() != 6) ++fails;
    for (std::size_t g = 0; g < rest.stats.size() && g + 6 < all.stats.size(); ++g) {
      const auto &a = all.stats[g + 6], &b = rest.stats[g];
      if (a.generation != b.generation || a.best != b.best || a.mean != b.mean || a.best_index != b.best_index ||
          a.species_sizes != b.species_sizes) { std::printf("resumed generation %zu differs\n", g); ++fails; }
    }
    if (!(all.best == rest.best) || !same_bits(full.population().pop_nodes, resumed.population().pop_nodes) ||
        !same_bits(full.population().pop_conns, resumed.population().pop_conns)) {
      std::printf("resumed population differs\n");
      ++fails;
    }
  }

  std::printf(fails ? "gpu.hpp parity FAILED (%d)\n" : "gpu.hpp parity ok\n", fails);
  return fails ? 1 : 0;
}
