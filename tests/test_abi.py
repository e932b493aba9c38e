"""CPU-side checks of the C ABI and host logic (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np

import oracle_lib as ol

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "flatneat_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fnb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2504_08339_b200 import _native
    lib = _native.lib()
    declared = _declared_symbols()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"{name} missing from the ctypes signature table"
    assert lib.fnb_abi_version() == 1


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        return
    import paper_2504_08339_b200 as fnb
    try:
        fnb.Engine(fnb.GenomeLimits(16, 32), [0, 1], [2])
    except fnb.FlatneatError as e:
        assert e.code == "eval_error"
    else:
        raise AssertionError("context creation must fail without a GPU")


def test_struct_layouts_match_oracle():
    from paper_2504_08339_b200 import _native as N
    assert C.sizeof(N.fnb_shape) == C.sizeof(ol.Shape)
    assert C.sizeof(N.fnb_schema) == C.sizeof(ol.Schema)
    assert C.sizeof(N.fnb_mutation_config) == C.sizeof(ol.MutCfg)


def test_synthetic_population_is_valid():
    from paper_2504_08339_b200.synthetic import synthetic_population
    nodes, conns = synthetic_population(64, 64, 256, fill=0.75, n_act=5, n_agg=4, seed=1)
    prob = ol.Problem(64, 256, [0, 1, 2, 3], [4])
    sh, sc = prob.c(), ol.RICH.c()
    buf = C.create_string_buffer(128)
    for i in range(64):
        n = np.ascontiguousarray(nodes[i])
        c = np.ascontiguousarray(conns[i])
        assert ol.oracle().fo_explain_invalid(C.byref(sh), C.byref(sc), ol.ptr(n, ol.F64P), ol.ptr(c, ol.F64P),
                                              buf, C.c_size_t(128)) == 0, buf.value
        t = ol.oracle_transform(prob, ol.RICH, n, c)
        assert t["status"] == 0 and t["order_count"] == 48
        assert int(np.sum(~np.isnan(c[:, 0]))) == 192


def test_python_innovation_table_mirrors_reference():
    """api.InnovationTable == ops.hpp:145-167: memo per generation, counter never runs back."""
    from paper_2504_08339_b200.api import InnovationTable
    t = InnovationTable(10)
    assert t.get_or_assign(1, 2) == 10 and t.get_or_assign(3, 4) == 11 and t.get_or_assign(1, 2) == 10
    t.reserve_up_to(5)
    assert t.next_key() == 12
    t.reserve_up_to(20)
    t.next_generation()
    assert t.get_or_assign(1, 2) == 20 and t.next_key() == 21
