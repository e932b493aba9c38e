/*
 * flatneat_b200.h -- C ABI of the B200-native NEAT generation loop.
 *
 * Drop-in boundary for the reference's header-only C++ API
 * (/root/reference/proj/include/flatneat/).  Plain pointers and sizes only,
 * no exceptions, no torch types.  Genomes cross the boundary in the
 * reference's own PopulationTensors layout (genome.hpp:315-338): P x N_max x 5
 * node rows [key,bias,response,agg_id,act_id] and P x C_max x 4 connection
 * rows [in,out,enabled,weight], FP64, NaN-padded.
 *
 * Status: every function returns 0 on success or 1 + Errc (errors.hpp:10-31);
 * fnb_last_error() then returns the reference's what() string
 * "<errc_name>: <detail>" and fnb_last_error_index() the lowest failing
 * genome (the lowest-chunk rule of parallel.hpp:69-73,108-109).
 *
 * Two layers:
 *   host layer   (fnb_transform, fnb_batch_forward, fnb_evaluate, ...)
 *                synchronous, host buffers in and out -- mirrors the reference
 *                free functions one for one;
 *   device layer (fnb_*_d) asynchronous on a caller stream, device pointers
 *                -- what the generation loop and multi-GPU driver compose.
 * A context owns one device and is not thread-safe (one host thread per ctx).
 */
#ifndef FLATNEAT_B200_H
#define FLATNEAT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FNB_ABI_VERSION 1
#define FNB_MAX_NODES_LIMIT 255   /* node rows fit a byte; row 255 is the forward's zero row */

/* Errc (errors.hpp:10-31); status = 1 + code. */
enum fnb_errc {
  FNB_E_UNKNOWN_FUNCTION = 0, FNB_E_GENOME_FULL, FNB_E_DUPLICATE_KEY,
  FNB_E_DUPLICATE_CONN, FNB_E_DANGLING_ENDPOINT, FNB_E_KEY_NOT_FOUND,
  FNB_E_PROTECTED_NODE, FNB_E_ATTR_OUT_OF_RANGE, FNB_E_SHAPE_MISMATCH,
  FNB_E_CORRUPT_ROW, FNB_E_CYCLE_DETECTED, FNB_E_NON_FINITE_INPUT,
  FNB_E_NON_FINITE_STATE, FNB_E_EMPTY_AGGREGATION, FNB_E_EMPTY_DATASET,
  FNB_E_PARSE_ERROR, FNB_E_VERSION_UNSUPPORTED, FNB_E_LIMITS_TOO_SMALL,
  FNB_E_CONFIG_ERROR, FNB_E_EVAL_ERROR
};

/* Built-in node functions (functions.hpp:17-21, 32). */
enum fnb_act { FNB_ACT_IDENTITY = 0, FNB_ACT_TANH, FNB_ACT_SIGMOID, FNB_ACT_RELU, FNB_ACT_SIN };
enum fnb_agg { FNB_AGG_SUM = 0, FNB_AGG_PRODUCT, FNB_AGG_MAX, FNB_AGG_MEAN };

/* Fitness epilogues fused into the forward. */
enum fnb_fitness {
  FNB_FIT_NONE = 0,          /* outputs only                                 */
  FNB_FIT_NEG_MSE = 1,       /* func-fit: -(1/(B*O)) sum (y - o)^2           */
  FNB_FIT_OFFSET_SSE = 2     /* xor:      offset - sum (y - o)^2             */
};

/* GenomeLimits + input/output keys (genome.hpp:87-92, 151-152). */
typedef struct fnb_shape {
  int max_nodes;
  int max_conns;
  int num_inputs;
  int num_outputs;
  const int* input_keys;
  const int* output_keys;
} fnb_shape;

/* AttributeSchema (genome.hpp:42-85) with names resolved to built-in codes. */
typedef struct fnb_schema {
  int n_act; int act[8];
  int n_agg; int agg[8];
  int default_act, default_agg;
} fnb_schema;

/* AttrMutation / MutationConfig / DistanceConfig (ops.hpp:117-140). */
typedef struct fnb_attr_mutation {
  double init_mean, init_std, mutate_power, mutate_rate, replace_rate;
} fnb_attr_mutation;

typedef struct fnb_mutation_config {
  double node_add, node_delete, conn_add, conn_delete;
  fnb_attr_mutation bias, response, weight;
  double activation_replace_rate, aggregation_replace_rate;
} fnb_mutation_config;

typedef struct fnb_distance_config {
  double compatibility_disjoint, compatibility_homologous;
} fnb_distance_config;

/* NeatConfig (Table 4 / Appendix C defaults in the Python
 * mirror).  Input keys must be 0..I-1 and output keys I..I+O-1. */
typedef struct fnb_neat_config {
  int pop_size;
  int max_species;              /* <= 32 */
  double compatibility_threshold;
  int species_elitism;
  int max_stagnation;
  int genome_elitism;
  double survival_threshold;
  double spawn_number_change_rate;
  int output_activation;        /* registry id given to output nodes at init */
  fnb_mutation_config mutation;
  fnb_distance_config distance;
} fnb_neat_config;

typedef struct fnb_ctx fnb_ctx;
typedef struct fnb_evolver fnb_evolver;

/* ---- context --------------------------------------------------------- */
int fnb_abi_version(void);
int fnb_ctx_create(const fnb_shape* shape, const fnb_schema* schema, int device, fnb_ctx** out);
void fnb_ctx_destroy(fnb_ctx* ctx);
const char* fnb_last_error(const fnb_ctx* ctx);
int fnb_last_error_index(const fnb_ctx* ctx);
/* bytes of one transformed network in the device net buffer */
size_t fnb_net_bytes(const fnb_ctx* ctx);
/* number of kernel launches this context issued since creation */
long long fnb_launch_count(const fnb_ctx* ctx);
/* tuning knob: sample columns per thread of the forward kernel (1, 2 or 4;
 * 0 = automatic).  Process-wide; results do not depend on it beyond FP32
 * summation order, which it does not change. */
void fnb_set_forward_spt(int spt);
/* tuning knobs of the forward launch geometry (process-wide; 0 = default):
 * spt columns per thread (1/2/4), max_cols sample columns per genome group
 * (power of two, default 128), rows_pct main-pass value-slot capacity in % of
 * max_nodes + 1 (default 62), group_kb shared-memory budget per genome group
 * (default 72).  Fitness bits do not depend on any of them. */
void fnb_set_forward_tuning(int spt, int max_cols, int rows_pct, int group_kb);
/* main-pass record capacity in % of the most records a genome can have
 * (default set in forward.cu); genomes with more records run in the overflow
 * pass.  Process-wide; fitness bits do not depend on it. */
void fnb_set_forward_recs_pct(int pct);
/* host-buffer transfer format of fnb_evaluate / fnb_batch_forward
 * (process-wide): 1 (default) packs the FP64 rows of PAGEABLE host arrays on
 * the host threads into the transfer rows K1 reads (0.40 of the bytes at C2,
 * converted exactly as K1 converts the FP64 rows) instead of staging them
 * whole; 0 stages and sends the FP64 rows.  Pinned arrays are sent as they are
 * either way.  Results are identical. */
void fnb_set_host_transfer_packed(int on);

/* ---- host layer (synchronous) ------------------------------------------ */

/* transform() over a population (network.hpp:122-220).  order_out: P*max_nodes
 * int32 rows, -1 padded (network.hpp:32); either output may be NULL. */
int fnb_transform(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P,
                  int32_t* order_out, int32_t* order_count_out);

/* transform() + batch_forward() (network.hpp:294-330): out[P][B][O].
 * inputs[B][I] sample-major like the reference; computed in FP32. */
int fnb_batch_forward(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P,
                      const double* inputs, int batch, double* out);

/* transform + forward + fused fitness epilogue -> fitness[P] (FP64). */
int fnb_evaluate(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P,
                 const double* inputs, const double* targets, int batch, int fitness_kind,
                 double fitness_offset, double* fitness_out);

/* distance() (ops.hpp:415-473) of every genome against S representatives:
 * out[P][S] = distance(genome_p, rep_s), FP64, bit-exact. */
int fnb_distance(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P,
                 const double* rep_nodes, const double* rep_conns, int S,
                 const fnb_distance_config* cfg, double* out);

/* crossover() (ops.hpp:382-407) of n parent pairs; keys[n][4] are RngKey
 * words (rng.hpp:44-72).  child_* receive n genomes. */
int fnb_crossover(fnb_ctx* ctx, const double* fit_nodes, const double* fit_conns,
                  const double* other_nodes, const double* other_conns, int n, const uint32_t* keys,
                  double* child_nodes, double* child_conns);

/* mutate() (ops.hpp:363-374) of P genomes in slot order with ONE
 * InnovationTable starting at *next_key (the population pattern of
 * ops.hpp:169-175), in place; keys[P][4] RngKey words.  On return *next_key
 * is the table's next key.  On error genomes below the failing index are
 * mutated and the rest untouched, as a sequential loop would leave them. */
int fnb_mutate(fnb_ctx* ctx, double* pop_nodes, double* pop_conns, int P, const uint32_t* keys,
               const fnb_mutation_config* cfg, int* next_key);

/* InnovationTable::get_or_assign of the caller's table (ops.hpp:149-156). */
typedef int (*fnb_innovation_fn)(void* user, int in_key, int out_key);
/* mutate() of P genomes in slot order against the caller's own table
 * (ops.hpp:169-175): `assign` is called once per splitting slot, in slot
 * order, exactly as the sequential loop calls get_or_assign, and the keys it
 * returns go into the genomes.  splits[P][3] (may be NULL) receives
 * (in_key, out_key, new_key) per slot, -1 for a slot that did not split.  A
 * duplicate_key failure at slot b (the key already names a node of genome b,
 * ops.hpp:19-23) leaves genomes [0, b) mutated, b.. untouched, and the table
 * with the calls up to and including b's. */
int fnb_mutate_table(fnb_ctx* ctx, double* pop_nodes, double* pop_conns, int P, const uint32_t* keys,
                     const fnb_mutation_config* cfg, fnb_innovation_fn assign, void* user, int32_t* splits);

/* RngKey(seed) and RngKey::split (rng.hpp:48-66), host side. */
void fnb_key_seed(uint64_t seed, uint32_t out[4]);
void fnb_key_split(const uint32_t key[4], uint64_t index, uint32_t out[4]);

/* ---- device layer (asynchronous on `stream`, device pointers) ------------ */

/* K3: d_out[P][S]. */
int fnb_distance_d(fnb_ctx* ctx, const double* d_nodes, const double* d_conns, int P,
                   const double* d_rep_nodes, const double* d_rep_conns, int S,
                   const fnb_distance_config* cfg, double* d_out, void* stream);
/* K5: child c = crossover(pop[fit[c]], pop[other[c]], keys[c]). */
int fnb_crossover_d(fnb_ctx* ctx, const double* d_nodes, const double* d_conns, const int32_t* d_fit,
                    const int32_t* d_other, const uint32_t* d_keys, int n, double* d_child_nodes,
                    double* d_child_conns, void* stream);
/* K6+K7: mutate P genomes in place (child c uses keys[c]); d_active[c] = 0
 * skips a child (elites; NULL = all).  d_next_key: 2 ints, [0] is the
 * InnovationTable counter (advanced in place), [1] scratch.  d_status[P]
 * receives 0 or 1 + Errc per child.  d_new_key[P] (may be NULL) receives the
 * key handed to each splitting child. */
int fnb_mutate_d(fnb_ctx* ctx, double* d_nodes, double* d_conns, int P, const uint32_t* d_keys,
                 const uint8_t* d_active, const fnb_mutation_config* cfg, int* d_next_key, int* d_status,
                 int* d_new_key, void* stream);
/* Sequential RngStream draws per key (parity tooling): kind 0 next_u64,
 * 1 uniform() bits, 2 below(n), 3 normal(0, 1) bits (rng.hpp:111-116, glibc
 * log / cos restated on the device).  d_out[n_keys][n_draws]. */
int fnb_stream_draws_d(fnb_ctx* ctx, const uint32_t* d_keys, int n_keys, int n_draws, int kind,
                       uint64_t n, uint64_t* d_out, void* stream);
/* d_out[i] = key.split(base + i), i < n (RngKey tree on the device). */
int fnb_split_keys_d(fnb_ctx* ctx, const uint32_t key[4], uint64_t base, int n, uint32_t* d_out,
                     void* stream);

/* K1: d_nets must hold P * fnb_net_bytes(ctx) bytes. */
int fnb_transform_d(fnb_ctx* ctx, const double* d_nodes, const double* d_conns, int P,
                    void* d_nets, void* stream);
/* Copy the int32 topological order (network.hpp:32) out of the net buffer. */
int fnb_net_order_d(fnb_ctx* ctx, const void* d_nets, int P, int32_t* d_order,
                    int32_t* d_order_count, void* stream);
/* Lowest failing genome (or -1) and its status; synchronises `stream` and
 * fills fnb_last_error() with the reference-format message. */
int fnb_check_nets_d(fnb_ctx* ctx, const double* d_nodes, const double* d_conns,
                     const void* d_nets, int P, void* stream);
/* K2: forward of P nets over X[B][I] (FP32); Y[B][O] targets for the fitness
 * epilogue; d_out (P*B*O doubles) and d_fitness (P doubles) may be NULL. */
int fnb_forward_d(fnb_ctx* ctx, const void* d_nets, int P, const float* d_X, const float* d_Y,
                  int batch, int fitness_kind, double fitness_offset, double* d_fitness,
                  double* d_out, void* stream);

/* ---- explain_invalid (genome.hpp:364-417) over a population ----------------
 * codes[p] = 0 for a valid genome, else the first failing check in the
 * reference's order (1-4 node row: partially NaN / non-integral key / bad
 * aggregation id / bad activation id, 5 duplicate node key, 6 input key
 * missing, 7 output key missing, 8-11 conn row: partially NaN / non-boolean
 * enabled flag / non-integral endpoint / missing node, 12 duplicate pair);
 * details[p] the row or key the message names.  fnb_explain_message formats
 * the reference's string ("" for 0) and returns its length. */
int fnb_explain_invalid(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P, int32_t* codes,
                        int32_t* details);
int fnb_explain_invalid_d(fnb_ctx* ctx, const double* d_nodes, const double* d_conns, int P, int32_t* d_codes,
                          int32_t* d_details, void* stream);
int fnb_explain_message(int code, int detail, char* buf, size_t n);

/* ---- BASELINE config 4: HyperNEAT ---------------------
 * The context's genomes are CPPNs with 5 inputs (x1, y1, x2, y2, bias) and 1
 * output.  Each CPPN is queried at the (num_obs + 1) x num_act substrate
 * connections (query q = j * (num_obs + 1) + i), its outputs become policy
 * weights (clamp to [-1, 1], |y| < weight_threshold -> 0, else rescaled to
 * max_weight), and the policy a = tanh(W [s, 1]) drives s' = A s + B a for
 * `steps` steps from s0; fitness = mean reward
 * -(|s'|^2 / num_obs) - act_cost |a|^2 / num_act.  A is num_obs x num_obs,
 * B num_obs x num_act (row-major); dynamics run in FP32, reward sums in FP64.
 * No reference code exists for this config: oracle/hyperneat.c
 * is the repo's FP64 restatement. */
typedef struct fnb_hyper_config {
  int num_obs, num_act, steps;        /* num_obs <= 31, num_act <= 32 */
  double weight_threshold, max_weight, act_cost;
} fnb_hyper_config;
/* host layer: genomes and dynamics from host memory; weights_out
 * ([P][num_act][num_obs+1] floats) may be NULL */
int fnb_hyper_evaluate(fnb_ctx* ctx, const double* pop_nodes, const double* pop_conns, int P,
                       const fnb_hyper_config* cfg, const double* A, const double* B, const double* s0,
                       double* fitness_out, float* weights_out);
/* device layer: transformed CPPNs (fnb_transform_d), FP32 dynamics on the device */
int fnb_hyper_evaluate_d(fnb_ctx* ctx, const void* d_nets, int P, const fnb_hyper_config* cfg, const float* d_A,
                         const float* d_B, const float* d_s0, double* d_fitness, float* d_weights, void* stream);

/* ---- the generation loop (PAPER Algorithm 1) -------------
 * An evolver owns a device-resident population of cfg->pop_size genomes, the
 * species state (<= 32 species), the fitness vector and the innovation
 * counter.  Semantics are the frozen restatement oracle/evolution.c (rules
 * E1-E5 in DESIGN.md): evaluate -> step (speciate, update_stagnation,
 * compute_spawn_counts, reproduce) -> next generation. */
int fnb_evolver_create(fnb_ctx* ctx, const fnb_neat_config* cfg, uint64_t seed, fnb_evolver** out);
void fnb_evolver_destroy(fnb_evolver* ev);  /* before fnb_ctx_destroy of its context */
int fnb_evolver_init_population(fnb_evolver* ev);  /* initialize_population */
/* set / get accept host or device pointers (unified addressing) */
int fnb_evolver_set_population(fnb_evolver* ev, const double* pop_nodes, const double* pop_conns);
int fnb_evolver_get_population(fnb_evolver* ev, double* pop_nodes, double* pop_conns);
int fnb_evolver_set_fitness(fnb_evolver* ev, const double* fitness);  /* inject (parity tests) */
int fnb_evolver_get_fitness(fnb_evolver* ev, double* fitness);
/* transform + forward + fitness of the current population */
int fnb_evolver_evaluate(fnb_evolver* ev, const double* inputs, const double* targets, int batch,
                         int fitness_kind, double fitness_offset);
int fnb_evolver_evaluate_d(fnb_evolver* ev, const float* d_X, const float* d_Y, int batch, int fitness_kind,
                           double fitness_offset);
/* The *_d evaluations are asynchronous: fnb_evolver_eval_check synchronises
 * the evolver stream and returns the last evaluation's error in the
 * reference's order -- the lowest genome whose transform failed (its
 * reference message, fnb_last_error_index = genome), else
 * non_finite_input (network.hpp:245-246).  batch <= 0 is empty_dataset
 * (SPEC.md:457).  The host variant fnb_evolver_evaluate checks itself. */
int fnb_evolver_eval_check(fnb_evolver* ev);
/* a rank's shard [lo, hi): fitness of those genomes into d_fitness_out[hi-lo] */
int fnb_evolver_evaluate_range_d(fnb_evolver* ev, int lo, int hi, const float* d_X, const float* d_Y, int batch,
                                 int fitness_kind, double fitness_offset, double* d_fitness_out);
/* device-to-device fitness injection (ordered on the evolver stream) */
int fnb_evolver_set_fitness_d(fnb_evolver* ev, const double* d_fitness);
/* population checksum (nodes, conns as 64-bit words: sum w_i*(2i+1) mod 2^64,
   xor next_key << 32, xor generation): replicas of one run agree bit for bit */
int fnb_evolver_checksum(fnb_evolver* ev, uint64_t* out);
int fnb_evolver_step(fnb_evolver* ev);
/* The same step split for sharded reproduction (one process per GPU, the
 * population replicated): every rank runs step_front (speciate, stagnation,
 * spawn, parent selection, node-split plans and innovation keys for ALL
 * slots), then step_back for its slot range [lo, hi) (crossover + mutation
 * into the next population buffer), the ranks all-gather the next buffer
 * (fnb_evolver_next_population), and every rank calls step_commit.  Slots
 * are independent, so the result equals fnb_evolver_step bit for bit. */
/* ---- the step sharded over ranks (distributed.py) -------------
 * Rank r of `world` owns genomes [bounds[r], bounds[r+1]) of the population
 * (evaluation, speciation distances, its children); the population buffers
 * keep global genome indices.  The caller runs the phases in order and, in
 * between, the collectives on the buffers fnb_evolver_shard_buffers names
 * (all exact: integer sums, MIN / MAX of integers or order-preserving bits,
 * broadcasts and all-gathers of bits), on the evolver's stream:
 *   all-gather fitness[lo,hi) -> fitness (each rank evaluates its shard)
 *   BEGIN                       first match against the old representatives
 *   repeat while species < max_species:
 *     MIN_UNASSIGNED            -> all-reduce MIN min_unassigned; f = its value
 *                                  (stop when INT_MAX); j = species count
 *     FOUND(a = f, b = j)       the owner of f writes representative slot j
 *                               -> broadcast rep slot j from f's owner
 *     JOIN(b = j)               commit species j, join the shard's genomes
 *   ASSIGN_REST                 nearest overflow -> all-reduce MIN rep_dmin
 *   REP_ARGMIN                  -> all-reduce MIN rep_argmin
 *   REP_STAGE                   -> all-reduce SUM rep_stage (u64 words)
 *   REP_COMMIT                  -> all-reduce SUM species_size
 *   COMPACT                     -> all-reduce MAX species_max
 *   STAGNATION                  -> all-reduce SUM rank_sum, rank_count;
 *                                  all-gather species_of[lo,hi) -> species_of
 *   SELECT(out = counts[world]) parents each rank holds (synchronises);
 *                               M = max(counts)
 *   PACK(a = M)                 -> all-gather send_* (M genomes) -> pool_*
 *   BACK(a = M)                 the shard's children -> all-reduce MIN first_bad
 *   fnb_evolver_step_commit
 * With world = 1 the sequence equals fnb_evolver_step bit for bit. */
enum fnb_shard_phase {
  FNB_SHARD_BEGIN = 0, FNB_SHARD_MIN_UNASSIGNED, FNB_SHARD_FOUND, FNB_SHARD_JOIN, FNB_SHARD_ASSIGN_REST,
  FNB_SHARD_REP_ARGMIN, FNB_SHARD_REP_STAGE, FNB_SHARD_REP_COMMIT, FNB_SHARD_COMPACT, FNB_SHARD_STAGNATION,
  FNB_SHARD_SELECT, FNB_SHARD_PACK, FNB_SHARD_BACK
};
typedef struct fnb_shard_buffers {
  int* min_unassigned;              /* 1                     MIN  */
  unsigned long long* rep_dmin;     /* 32                    MIN  */
  int* rep_argmin;                  /* 32                    MIN  */
  unsigned long long* rep_stage;    /* rep_stage_words       SUM  */
  size_t rep_stage_words;
  int* species_size;                /* 32                    SUM  */
  unsigned long long* species_max;  /* 32                    MAX  */
  long long* rank_sum;              /* 32                    SUM  */
  int* rank_count;                  /* 32                    SUM  */
  int* first_bad;                   /* 1                     MIN  */
  double* fitness;                  /* pop_size              all-gather */
  int* species_of;                  /* pop_size              all-gather */
  double* rep_nodes;                /* 32 genomes            broadcast of one slot */
  double* rep_conns;
  double* send_nodes;               /* M genomes (after PACK) */
  double* send_conns;
  double* pool_nodes;               /* world x M genomes     all-gather of send_* */
  double* pool_conns;
} fnb_shard_buffers;
int fnb_evolver_shard_init(fnb_evolver* ev, int world, const int* bounds);
/* species count before the next step (host mirror; no synchronisation) */
int fnb_evolver_host_species(fnb_evolver* ev);
int fnb_evolver_shard_buffers(fnb_evolver* ev, fnb_shard_buffers* out);
int fnb_evolver_shard_phase(fnb_evolver* ev, int phase, int rank, int a, int b, int* out);

/* explain_invalid over the current population: first_invalid = lowest invalid
 * genome or -1; an invalid one also returns 1 + FNB_E_CORRUPT_ROW with the
 * reference's explanation in fnb_last_error */
int fnb_evolver_validate(fnb_evolver* ev, int* first_invalid);
int fnb_evolver_step_front(fnb_evolver* ev);
int fnb_evolver_step_back(fnb_evolver* ev, int lo, int hi);
int fnb_evolver_step_commit(fnb_evolver* ev);
int fnb_evolver_next_population(fnb_evolver* ev, double** d_nodes, double** d_conns);
/* species arrays have room for 32 entries; species_of[pop_size] may be NULL */
int fnb_evolver_species(fnb_evolver* ev, int* count, int* ids, int* sizes, int* spawn, double* best,
                        int* stagnation, int* species_of);
int fnb_evolver_state(fnb_evolver* ev, int* generation, int* next_key);
/* InnovationTable::reserve_up_to for a population loaded with set_population */
int fnb_evolver_set_next_key(fnb_evolver* ev, int next_key);
/* ---- checkpoint / resume ---------------------------------------------------
 * Everything a generation step reads besides the population (SPEC.md:337-340
 * SpeciesState; the key tree root of oracle E1): after set_population with
 * the saved population and set_state with the saved record and
 * representatives, the run continues bit for bit. */
typedef struct fnb_run_state {
  uint64_t seed;                /* RngKey(seed) root of the key tree          */
  int generation;               /* generations stepped so far                 */
  int next_key;                 /* InnovationTable counter (ops.hpp:145-167)  */
  int species_count;
  int next_species_id;
  int species_id[32];           /* ascending                                   */
  double species_best[32];      /* best-ever fitness                           */
  int species_stagnation[32];
  int species_size[32];         /* members at the last speciation              */
  int species_spawn[32];
} fnb_run_state;
/* rep_nodes [species_count][max_nodes][5], rep_conns [species_count][max_conns][4]
 * (either may be NULL on get) */
int fnb_evolver_get_state(fnb_evolver* ev, fnb_run_state* state, double* rep_nodes, double* rep_conns);
int fnb_evolver_set_state(fnb_evolver* ev, const fnb_run_state* state, const double* rep_nodes,
                          const double* rep_conns);

/* ---- SPEC evolve(problem, cfg, key) ------------------------
 * RunStats: one record per completed generation. */
typedef struct fnb_run_stats {
  int generation;               /* the evolver's generation counter at evaluation */
  double best, mean, std;       /* fitness over the population (population std) */
  int best_index;               /* argmax, lowest index on ties                */
  int species_count;            /* after this generation's speciation          */
  int species_size[32];
  double elapsed_ms;            /* wall clock of the generation                */
} fnb_run_stats;
/* called after every generation; a nonzero return stops the run */
typedef int (*fnb_run_stats_fn)(void* user, const fnb_run_stats* stats);
/* Loops evaluate -> (stop if best >= fitness_target) -> step for at most
 * generation_limit generations on the func-fit / xor problem given by
 * inputs[batch][I], targets[batch][O] and fitness_kind; each generation runs
 * as one CUDA graph with the termination test on the device.  Returns
 * pop[argmax(fit)] of the last evaluated generation (best_* may be NULL).
 * Evaluation errors abort with "generation g, genome i: ..." context
 * (SPEC.md:419). */
int fnb_evolve(fnb_evolver* ev, const double* inputs, const double* targets, int batch, int fitness_kind,
               double fitness_offset, double fitness_target, int generation_limit, fnb_run_stats_fn on_generation,
               void* user, double* best_nodes, double* best_conns, double* best_fitness, int* generations_run);
/* how the last fnb_evolve ran: 2 one graph per generation (conditional step
 * node), 1 evaluate graph + host check + step graph, 0 eager; -1 never ran */
int fnb_evolver_run_mode(fnb_evolver* ev);

/* device pointers of the current population / fitness and the evolver's stream */
int fnb_evolver_device_state(fnb_evolver* ev, double** d_nodes, double** d_conns, double** d_fitness,
                             void** stream);

#ifdef __cplusplus
}
#endif
#endif /* FLATNEAT_B200_H */
