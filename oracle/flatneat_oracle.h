/*
 * flatneat_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C (C11) restatement of the reference flatneat CPU path
 * (/root/reference/proj/include/flatneat/ *.hpp) plus a restatement of the
 * SPEC-only evolution module that the reference never
 * implemented.  It exists to CHECK the CUDA path; nothing in the product
 * (paper_2504_08339_b200/) may link, import or call it.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
 *
 * Parity pinning:
 *   - Every function below that restates reference code is pinned against
 *     the reference itself, compiled from /root/reference by
 *     oracle/Makefile into oracle/_ref/libflatneat_ref.so
 *     (tests/test_oracle_vs_ref.py), and against golden vectors dumped from
 *     that library (tests/golden/).
 *   - The evolution restatement (fo_speciate ... fo_reproduce) has no
 *     reference code: "parity unpinned" for those stages;
 *     it is frozen by tests/golden/evolution_*.
 *
 * Conventions: genomes are the reference's NaN-padded FP64 rows
 * (node row [key,bias,response,agg_id,act_id], conn row [in,out,enabled,w],
 * genome.hpp:19-38).  Status returns are 0 for success or 1 + Errc
 * (errors.hpp:10-31).  The build uses no -march and -ffp-contract=off so
 * FP64 arithmetic rounds exactly like the reference's Release build
 * (CMakeLists.txt:4-9: no FMA contraction).
 */
#ifndef FLATNEAT_ORACLE_H
#define FLATNEAT_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  FO_NODE_COLS = 5, FO_CONN_COLS = 4,
  FO_NODE_KEY = 0, FO_NODE_BIAS = 1, FO_NODE_RESP = 2, FO_NODE_AGG = 3, FO_NODE_ACT = 4,
  FO_CONN_IN = 0, FO_CONN_OUT = 1, FO_CONN_EN = 2, FO_CONN_W = 3
};

/* Errc numbering (errors.hpp:10-31). Status = 1 + code. */
enum {
  FO_E_unknown_function = 0, FO_E_genome_full, FO_E_duplicate_key,
  FO_E_duplicate_conn, FO_E_dangling_endpoint, FO_E_key_not_found,
  FO_E_protected_node, FO_E_attr_out_of_range, FO_E_shape_mismatch,
  FO_E_corrupt_row, FO_E_cycle_detected, FO_E_non_finite_input,
  FO_E_non_finite_state, FO_E_empty_aggregation, FO_E_empty_dataset,
  FO_E_parse_error, FO_E_version_unsupported, FO_E_limits_too_small,
  FO_E_config_error, FO_E_eval_error
};

/* Built-in functions (functions.hpp:17-21, 32). */
enum { FO_ACT_IDENTITY = 0, FO_ACT_TANH, FO_ACT_SIGMOID, FO_ACT_RELU, FO_ACT_SIN };
enum { FO_AGG_SUM = 0, FO_AGG_PRODUCT, FO_AGG_MAX, FO_AGG_MEAN };

/* ---- RNG: rng.hpp:19-134 ------------------------------------------------ */
typedef struct { uint32_t w[4]; } fo_key;
typedef struct {
  fo_key key;
  uint64_t block;
  uint32_t buf[4];
  int avail;
} fo_stream;

void fo_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
fo_key fo_key_seed(uint64_t seed);
fo_key fo_key_split(fo_key k, uint64_t index);
void fo_stream_init(fo_stream* s, fo_key k);
uint64_t fo_next_u64(fo_stream* s);
double fo_uniform(fo_stream* s);
int fo_coin(fo_stream* s, double p);
uint64_t fo_below(fo_stream* s, uint64_t n);
double fo_normal(fo_stream* s, double mean, double sd);

/* ---- Shapes ------------------------------------------------------------- */
typedef struct {
  int max_nodes, max_conns;
  int num_inputs, num_outputs;
  const int* input_keys;   /* num_inputs  */
  const int* output_keys;  /* num_outputs */
} fo_shape;

typedef struct {
  int n_act; int act[8];     /* registry id -> FO_ACT_* */
  int n_agg; int agg[8];     /* registry id -> FO_AGG_* */
  int default_act, default_agg;
} fo_schema;

/* ---- Transform / forward: network.hpp:122-330 --------------------------- */
typedef struct {
  /* outputs, caller-allocated */
  int32_t* order;        /* max_nodes, -1 tail */
  int order_count;
  int* in_begin;         /* max_nodes+1: CSR over dst rows */
  int* in_src;           /* max_conns: src rows, ascending per dst */
  double* in_w;          /* max_conns */
  int* input_rows;       /* num_inputs */
  int* output_rows;      /* num_outputs */
  /* error detail */
  char msg[512];
} fo_net;

int fo_transform(const fo_shape* sh, const fo_schema* sc, const double* nodes,
                 const double* conns, fo_net* net);
int fo_forward(const fo_shape* sh, const fo_schema* sc, const double* nodes,
               const fo_net* net, const double* inputs, double* outputs,
               double* scratch_values /* max_nodes */);

/* ---- Ops: ops.hpp ------------------------------------------------------- */
typedef struct { double init_mean, init_std, mutate_power, mutate_rate, replace_rate; } fo_attr_mut;
typedef struct {
  double node_add, node_delete, conn_add, conn_delete;
  fo_attr_mut bias, response, weight;
  double activation_replace_rate, aggregation_replace_rate;
} fo_mut_cfg;
typedef struct { double compatibility_disjoint, compatibility_homologous; } fo_dist_cfg;

double fo_distance(const fo_shape* sh, const double* n1, const double* c1,
                   const double* n2, const double* c2, const fo_dist_cfg* cfg);
void fo_crossover(const fo_shape* sh, const double* fit_n, const double* fit_c,
                  const double* oth_n, const double* oth_c, fo_key key,
                  double* child_n, double* child_c);

typedef struct { int split; int in_key; int out_key; } fo_split_plan;
fo_split_plan fo_plan_node_split(const fo_shape* sh, const double* nodes,
                                 const double* conns, fo_key key, const fo_mut_cfg* cfg);
/* In-place on (nodes, conns).  Returns status. */
int fo_apply_node_split(const fo_shape* sh, const fo_schema* sc, double* nodes,
                        double* conns, fo_split_plan plan, int new_key,
                        fo_key key, const fo_mut_cfg* cfg);
int fo_mutate_rest(const fo_shape* sh, const fo_schema* sc, double* nodes,
                   double* conns, fo_key key, const fo_mut_cfg* cfg);

/* InnovationTable (ops.hpp:145-167): flat array map. */
typedef struct {
  int next_key;
  int count, cap;
  int* pairs;  /* 3*cap: in, out, key */
} fo_innov;
void fo_innov_init(fo_innov* t, int first_key);
void fo_innov_free(fo_innov* t);
int fo_innov_get_or_assign(fo_innov* t, int in_key, int out_key);
void fo_innov_next_generation(fo_innov* t);

/* Whole mutate (ops.hpp:363-374), in place. */
int fo_mutate(const fo_shape* sh, const fo_schema* sc, double* nodes,
              double* conns, fo_key key, const fo_mut_cfg* cfg, fo_innov* t);

/* Structural primitives (ops.hpp:19-89), in place; return status. */
int fo_add_node(const fo_shape* sh, double* nodes, const double row[5]);
int fo_remove_node(const fo_shape* sh, double* nodes, double* conns, int key);
int fo_add_conn(const fo_shape* sh, const double* nodes, double* conns, const double row[4]);
int fo_remove_conn(const fo_shape* sh, double* conns, int in_key, int out_key);
int fo_creates_cycle(const fo_shape* sh, const double* conns, int from_key, int to_key);
int fo_explain_invalid(const fo_shape* sh, const fo_schema* sc, const double* nodes,
                       const double* conns, char* buf, size_t n);

/* Test generator (tests/support/generators.hpp:37-84) -> padded genome.
 * Returns status (genome_full if it does not fit). */
typedef struct { int num_inputs, num_outputs, max_hidden; double conn_prob, disabled_prob; } fo_genspec;
int fo_random_acyclic_genome(fo_stream* s, const fo_schema* sc, const fo_genspec* spec,
                             int max_nodes, int max_conns, double* nodes, double* conns);

/* ---- Evolution (no reference code: parity unpinned) --- */
typedef struct {
  int pop_size;
  int max_species;
  double compatibility_threshold;
  int species_elitism;
  int max_stagnation;
  int genome_elitism;
  double survival_threshold;
  double spawn_number_change_rate;
  int output_activation;   /* registry id for output nodes at init */
  fo_mut_cfg mutation;
  fo_dist_cfg distance;
} fo_neat_cfg;

typedef struct {
  int count;
  int next_id;
  int cap;
  size_t nsz, csz;         /* doubles per rep node / conn tensor */
  int* id;                 /* [cap] ascending */
  double* rep_nodes;       /* [cap * max_nodes*5] */
  double* rep_conns;       /* [cap * max_conns*4] */
  double* best_fitness;    /* [cap] best-ever */
  int* stagnation;         /* [cap] */
  int* size;               /* [cap] members this generation */
  int* spawn;              /* [cap] */
} fo_species;

void fo_species_init(fo_species* s, const fo_shape* sh, int cap);
void fo_species_free(fo_species* s);

/* Initial population. pop_nodes [P*N*5], pop_conns [P*C*4]. */
int fo_initialize_population(const fo_shape* sh, const fo_schema* sc,
                             const fo_neat_cfg* cfg, uint64_t seed,
                             double* pop_nodes, double* pop_conns);
/* speciate: writes species_of[P] (index into s after the
 * call) and updates representatives/sizes.  dist_scratch: P*(max_species) */
void fo_speciate(const fo_shape* sh, const fo_neat_cfg* cfg, const double* pop_nodes,
                 const double* pop_conns, fo_species* s, int* species_of);
/* update_stagnation: drops stale species in place and
 * remaps species_of (-1 = member of a removed species). */
void fo_update_stagnation(const fo_neat_cfg* cfg, const double* fitness,
                          fo_species* s, int* species_of);
/* compute_spawn_counts -> s->spawn */
void fo_compute_spawn(const fo_neat_cfg* cfg, const double* fitness,
                      const int* species_of, fo_species* s);
/* reproduce: writes the next population. */
int fo_reproduce(const fo_shape* sh, const fo_schema* sc, const fo_neat_cfg* cfg,
                 const double* pop_nodes, const double* pop_conns,
                 const double* fitness, const int* species_of,
                 const fo_species* s, uint64_t seed, int generation,
                 fo_innov* innov, double* next_nodes, double* next_conns,
                 int* parent_a, int* parent_b);

/* ---- HyperNEAT (BASELINE config 4; this repo's definition, hyperneat.c) -- */
typedef struct {
  int n_obs, n_act, steps;
  double weight_threshold, max_weight, act_cost;
} fo_hyper_cfg;
void fo_hyper_queries(const fo_hyper_cfg* c, double* q /* [(n_obs+1)*n_act][5] */);
double fo_hyper_weight(const fo_hyper_cfg* c, double cppn_out);
void fo_hyper_substrate(const fo_hyper_cfg* c, const double* cppn_out /* Q */, double* W /* [n_act][n_obs+1] */);
double fo_hyper_rollout(const fo_hyper_cfg* c, const double* W, const double* A, const double* B,
                        const double* s0);

#ifdef __cplusplus
}
#endif
#endif
