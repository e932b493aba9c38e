"""B200-native tensorized NEAT generation loop (TensorNEAT, arXiv 2504.08339).

The compute lives in libflatneat_b200.so (sm_100a CUDA kernels behind the C
ABI of include/flatneat_b200.h); this package is the host-side mirror of the
reference flatneat API.  Importing it without the built library fails loudly.
"""
from . import _native
from .api import (ACTIVATIONS, AGGREGATIONS, ERRC, FIT_NEG_MSE, FIT_NONE, FIT_OFFSET_SSE, AttrMutation,
                  AttributeSchema, BatchResult, DistanceConfig, Engine, FlatneatError, GenomeLimits,
                  HyperConfig, InnovationTable, MutationConfig, PopulationTensors)

_native.lib()  # fail at import time if the CUDA library is absent

__all__ = ["ACTIVATIONS", "AGGREGATIONS", "ERRC", "FIT_NEG_MSE", "FIT_NONE", "FIT_OFFSET_SSE", "AttrMutation",
           "AttributeSchema", "BatchResult", "DistanceConfig", "Engine", "FlatneatError", "GenomeLimits",
           "HyperConfig", "InnovationTable", "MutationConfig", "PopulationTensors"]
