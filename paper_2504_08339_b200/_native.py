"""ctypes binding of libflatneat_b200.so (include/flatneat_b200.h).

There is no fallback: if the CUDA library is missing or cannot be loaded,
importing the package fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libflatneat_b200.so")


class fnb_shape(C.Structure):
    _fields_ = [("max_nodes", C.c_int), ("max_conns", C.c_int), ("num_inputs", C.c_int),
                ("num_outputs", C.c_int), ("input_keys", C.POINTER(C.c_int)),
                ("output_keys", C.POINTER(C.c_int))]


class fnb_schema(C.Structure):
    _fields_ = [("n_act", C.c_int), ("act", C.c_int * 8), ("n_agg", C.c_int), ("agg", C.c_int * 8),
                ("default_act", C.c_int), ("default_agg", C.c_int)]


class fnb_attr_mutation(C.Structure):
    _fields_ = [("init_mean", C.c_double), ("init_std", C.c_double), ("mutate_power", C.c_double),
                ("mutate_rate", C.c_double), ("replace_rate", C.c_double)]


class fnb_mutation_config(C.Structure):
    _fields_ = [("node_add", C.c_double), ("node_delete", C.c_double), ("conn_add", C.c_double),
                ("conn_delete", C.c_double), ("bias", fnb_attr_mutation), ("response", fnb_attr_mutation),
                ("weight", fnb_attr_mutation), ("activation_replace_rate", C.c_double),
                ("aggregation_replace_rate", C.c_double)]


class fnb_distance_config(C.Structure):
    _fields_ = [("compatibility_disjoint", C.c_double), ("compatibility_homologous", C.c_double)]


class fnb_neat_config(C.Structure):
    _fields_ = [("pop_size", C.c_int), ("max_species", C.c_int), ("compatibility_threshold", C.c_double),
                ("species_elitism", C.c_int), ("max_stagnation", C.c_int), ("genome_elitism", C.c_int),
                ("survival_threshold", C.c_double), ("spawn_number_change_rate", C.c_double),
                ("output_activation", C.c_int), ("mutation", fnb_mutation_config),
                ("distance", fnb_distance_config)]


class fnb_hyper_config(C.Structure):
    _fields_ = [("num_obs", C.c_int), ("num_act", C.c_int), ("steps", C.c_int), ("weight_threshold", C.c_double),
                ("max_weight", C.c_double), ("act_cost", C.c_double)]


class fnb_run_state(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("generation", C.c_int), ("next_key", C.c_int), ("species_count", C.c_int),
                ("next_species_id", C.c_int), ("species_id", C.c_int * 32), ("species_best", C.c_double * 32),
                ("species_stagnation", C.c_int * 32), ("species_size", C.c_int * 32),
                ("species_spawn", C.c_int * 32)]


class fnb_run_stats(C.Structure):
    _fields_ = [("generation", C.c_int), ("best", C.c_double), ("mean", C.c_double), ("std", C.c_double),
                ("best_index", C.c_int), ("species_count", C.c_int), ("species_size", C.c_int * 32),
                ("elapsed_ms", C.c_double)]


class fnb_shard_buffers(C.Structure):
    _fields_ = [("min_unassigned", C.c_void_p), ("rep_dmin", C.c_void_p), ("rep_argmin", C.c_void_p),
                ("rep_stage", C.c_void_p), ("rep_stage_words", C.c_size_t), ("species_size", C.c_void_p),
                ("species_max", C.c_void_p), ("rank_sum", C.c_void_p), ("rank_count", C.c_void_p),
                ("first_bad", C.c_void_p), ("fitness", C.c_void_p), ("species_of", C.c_void_p),
                ("rep_nodes", C.c_void_p), ("rep_conns", C.c_void_p), ("send_nodes", C.c_void_p),
                ("send_conns", C.c_void_p), ("pool_nodes", C.c_void_p), ("pool_conns", C.c_void_p)]


# typedef int (*fnb_run_stats_fn)(void* user, const fnb_run_stats* stats)
RUN_STATS_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(fnb_run_stats))

VP = C.c_void_p
DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int32)
U32P = C.POINTER(C.c_uint32)

# name -> (restype, argtypes); every symbol include/flatneat_b200.h declares
SIGNATURES = {
    "fnb_abi_version": (C.c_int, []),
    "fnb_ctx_create": (C.c_int, [C.POINTER(fnb_shape), C.POINTER(fnb_schema), C.c_int, C.POINTER(VP)]),
    "fnb_ctx_destroy": (None, [VP]),
    "fnb_last_error": (C.c_char_p, [VP]),
    "fnb_last_error_index": (C.c_int, [VP]),
    "fnb_net_bytes": (C.c_size_t, [VP]),
    "fnb_launch_count": (C.c_longlong, [VP]),
    "fnb_set_forward_spt": (None, [C.c_int]),
    "fnb_set_forward_tuning": (None, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "fnb_set_forward_recs_pct": (None, [C.c_int]),
    "fnb_set_host_transfer_packed": (None, [C.c_int]),
    "fnb_transform": (C.c_int, [VP, DP, DP, C.c_int, IP, IP]),
    "fnb_batch_forward": (C.c_int, [VP, DP, DP, C.c_int, DP, C.c_int, DP]),
    "fnb_evaluate": (C.c_int, [VP, DP, DP, C.c_int, DP, DP, C.c_int, C.c_int, C.c_double, DP]),
    "fnb_transform_d": (C.c_int, [VP, VP, VP, C.c_int, VP, VP]),
    "fnb_net_order_d": (C.c_int, [VP, VP, C.c_int, VP, VP, VP]),
    "fnb_check_nets_d": (C.c_int, [VP, VP, VP, VP, C.c_int, VP]),
    "fnb_forward_d": (C.c_int, [VP, VP, C.c_int, VP, VP, C.c_int, C.c_int, C.c_double, VP, VP, VP]),
    "fnb_distance": (C.c_int, [VP, DP, DP, C.c_int, DP, DP, C.c_int, C.POINTER(fnb_distance_config), DP]),
    "fnb_crossover": (C.c_int, [VP, DP, DP, DP, DP, C.c_int, U32P, DP, DP]),
    "fnb_key_seed": (None, [C.c_uint64, U32P]),
    "fnb_key_split": (None, [U32P, C.c_uint64, U32P]),
    "fnb_distance_d": (C.c_int, [VP, VP, VP, C.c_int, VP, VP, C.c_int, C.POINTER(fnb_distance_config), VP, VP]),
    "fnb_crossover_d": (C.c_int, [VP, VP, VP, VP, VP, VP, C.c_int, VP, VP, VP]),
    "fnb_mutate": (C.c_int, [VP, DP, DP, C.c_int, U32P, C.POINTER(fnb_mutation_config), C.POINTER(C.c_int)]),
    "fnb_mutate_table": (C.c_int, [VP, DP, DP, C.c_int, U32P, C.POINTER(fnb_mutation_config), VP, VP, IP]),
    "fnb_evolver_eval_check": (C.c_int, [VP]),
    "fnb_evolver_get_state": (C.c_int, [VP, C.POINTER(fnb_run_state), DP, DP]),
    "fnb_evolver_set_state": (C.c_int, [VP, C.POINTER(fnb_run_state), DP, DP]),
    "fnb_evolver_run_mode": (C.c_int, [VP]),
    "fnb_evolver_host_species": (C.c_int, [VP]),
    "fnb_evolver_shard_init": (C.c_int, [VP, C.c_int, IP]),
    "fnb_evolver_shard_buffers": (C.c_int, [VP, C.POINTER(fnb_shard_buffers)]),
    "fnb_evolver_shard_phase": (C.c_int, [VP, C.c_int, C.c_int, C.c_int, C.c_int, IP]),
    "fnb_evolve": (C.c_int, [VP, DP, DP, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, VP, VP, DP, DP, DP,
                             C.POINTER(C.c_int)]),
    "fnb_mutate_d": (C.c_int, [VP, VP, VP, C.c_int, VP, VP, C.POINTER(fnb_mutation_config), VP, VP, VP, VP]),
    "fnb_evolver_create": (C.c_int, [VP, C.POINTER(fnb_neat_config), C.c_uint64, C.POINTER(VP)]),
    "fnb_evolver_destroy": (None, [VP]),
    "fnb_evolver_init_population": (C.c_int, [VP]),
    "fnb_evolver_set_population": (C.c_int, [VP, DP, DP]),
    "fnb_evolver_get_population": (C.c_int, [VP, DP, DP]),
    "fnb_evolver_set_fitness": (C.c_int, [VP, DP]),
    "fnb_evolver_get_fitness": (C.c_int, [VP, DP]),
    "fnb_evolver_evaluate": (C.c_int, [VP, DP, DP, C.c_int, C.c_int, C.c_double]),
    "fnb_evolver_evaluate_d": (C.c_int, [VP, VP, VP, C.c_int, C.c_int, C.c_double]),
    "fnb_evolver_step": (C.c_int, [VP]),
    "fnb_evolver_validate": (C.c_int, [VP, C.POINTER(C.c_int)]),
    "fnb_evolver_step_front": (C.c_int, [VP]),
    "fnb_evolver_step_back": (C.c_int, [VP, C.c_int, C.c_int]),
    "fnb_evolver_step_commit": (C.c_int, [VP]),
    "fnb_evolver_next_population": (C.c_int, [VP, C.POINTER(VP), C.POINTER(VP)]),
    "fnb_evolver_evaluate_range_d": (C.c_int, [VP, C.c_int, C.c_int, VP, VP, C.c_int, C.c_int, C.c_double, VP]),
    "fnb_evolver_set_fitness_d": (C.c_int, [VP, VP]),
    "fnb_evolver_checksum": (C.c_int, [VP, C.POINTER(C.c_uint64)]),
    "fnb_evolver_species": (C.c_int, [VP, IP, IP, IP, IP, DP, IP, IP]),
    "fnb_evolver_state": (C.c_int, [VP, IP, IP]),
    "fnb_evolver_set_next_key": (C.c_int, [VP, C.c_int]),
    "fnb_evolver_device_state": (C.c_int, [VP, C.POINTER(VP), C.POINTER(VP), C.POINTER(VP), C.POINTER(VP)]),
    "fnb_stream_draws_d": (C.c_int, [VP, VP, C.c_int, C.c_int, C.c_int, C.c_uint64, VP, VP]),
    "fnb_split_keys_d": (C.c_int, [VP, U32P, C.c_uint64, C.c_int, VP, VP]),
    "fnb_explain_invalid": (C.c_int, [VP, DP, DP, C.c_int, IP, IP]),
    "fnb_explain_invalid_d": (C.c_int, [VP, VP, VP, C.c_int, VP, VP, VP]),
    "fnb_explain_message": (C.c_int, [C.c_int, C.c_int, C.c_char_p, C.c_size_t]),
    "fnb_hyper_evaluate": (C.c_int, [VP, DP, DP, C.c_int, C.POINTER(fnb_hyper_config), DP, DP, DP, DP,
                                     C.POINTER(C.c_float)]),
    "fnb_hyper_evaluate_d": (C.c_int, [VP, VP, C.c_int, C.POINTER(fnb_hyper_config), VP, VP, VP, VP, VP, VP]),
}

# typedef int (*fnb_innovation_fn)(void* user, int in_key, int out_key)
INNOVATION_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int)

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(the CUDA library is required; there is no CPU fallback)")
        lib_ = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib_, name)
            f.restype = res
            f.argtypes = args
        _lib = lib_
    return _lib
