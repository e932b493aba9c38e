"""explain_invalid (genome.hpp:364-417) on the device (csrc/validate.cu)
against the reference's own function (oracle/_ref), string for string, on
valid genomes and on every kind of corruption the reference names."""
import numpy as np
import pytest

import oracle_lib as ol

pytestmark = pytest.mark.gpu

KINDS = ["node_partial", "node_key_frac", "node_key_neg", "node_agg", "node_act", "dup_key", "no_input",
         "no_output", "conn_partial", "conn_enabled", "conn_endpoint", "conn_missing", "dup_pair", "huge_endpoint",
         "late_partial_with_dup"]


@pytest.fixture(scope="module")
def fnb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_08339_b200 as m
    return m


def _corrupt(n, c, kind, rng):
    n, c = n.copy(), c.copy()
    live_n = np.where(~np.isnan(n[:, 0]))[0]
    live_c = np.where(~np.isnan(c[:, 0]))[0]
    hidden = [r for r in live_n if n[r, 0] > 3]
    r = int(rng.choice(live_n))
    if live_c.size == 0:  # give the genome one connection to corrupt
        c[0] = [0.0, 3.0, 1.0, 0.5]
        live_c = np.array([0])
    q = int(rng.choice(live_c))
    if kind == "node_partial": n[r, 2] = np.nan
    elif kind == "node_key_frac": n[r, 0] += 0.5
    elif kind == "node_key_neg": n[r, 0] = -3.0
    elif kind == "node_agg": n[r, 3] = 7.0
    elif kind == "node_act": n[r, 4] = 1.5
    elif kind == "dup_key": n[r, 0] = n[live_n[0], 0] if r != live_n[0] else n[live_n[-1], 0]
    elif kind == "no_input": n[0] = np.nan; c[(c[:, 0] == 0) | (c[:, 1] == 0)] = np.nan
    elif kind == "no_output": n[3] = np.nan; c[(c[:, 0] == 3) | (c[:, 1] == 3)] = np.nan
    elif kind == "conn_partial": c[q, 3] = np.inf
    elif kind == "conn_enabled": c[q, 2] = 0.5
    elif kind == "conn_endpoint": c[q, 1] += 0.25
    elif kind == "conn_missing": c[q, 0] = 999.0
    elif kind == "dup_pair":
        free = np.where(np.isnan(c[:, 0]))[0]
        c[free[0]] = c[q]
    elif kind == "huge_endpoint": c[q, 0] = 3e9   # int() of it is INT_MIN on x86: "non-integral endpoint"
    elif kind == "late_partial_with_dup":  # the node-row loop reports before duplicate keys
        if len(hidden) > 1:
            n[hidden[0], 0] = n[hidden[1], 0]
        n[live_n[-1], 1] = np.nan
    return n, c


def test_explain_invalid_matches_reference(fnb):
    schema = ol.SchemaSpec(["tanh", "sigmoid", "identity"], ["sum", "product"])
    prob = ol.Problem(20, 64, [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(404, schema, 60, 20, 64)
    rng = np.random.default_rng(8)
    pn, pc, kinds = [], [], []
    for i in range(nodes.shape[0]):
        kind = "valid" if i % 4 == 0 else KINDS[i % len(KINDS)]
        n, c = (nodes[i], conns[i]) if kind == "valid" else _corrupt(nodes[i], conns[i], kind, rng)
        pn.append(n)
        pc.append(c)
        kinds.append(kind)
    pn, pc = np.stack(pn), np.stack(pc)
    eng = fnb.Engine(fnb.GenomeLimits(20, 64), [0, 1, 2], [3], fnb.AttributeSchema(list(schema.activations),
                                                                                  list(schema.aggregations)))
    got = eng.explain_invalid(pn, pc)
    seen = set()
    for i in range(pn.shape[0]):
        want = ol.explain_invalid(prob, schema, pn[i], pc[i])
        assert got[i] == want, (i, kinds[i], got[i], want)
        seen.add(want.split(" ")[0] + (" " + want.split(" ")[-1] if want else ""))
    assert len(seen) >= 10  # the corruptions exercised most of the reference's messages


def test_evolver_population_stays_valid(fnb):
    """A device run validated after every generation (the SPEC's invariant
    that every genome the loop produces is valid)."""
    from paper_2504_08339_b200.evolve import Evolver, NeatConfig
    from paper_2504_08339_b200.synthetic import regression_dataset
    eng = fnb.Engine(fnb.GenomeLimits(24, 80), [0, 1, 2], [3], fnb.AttributeSchema(["tanh", "sigmoid"], ["sum"]))
    m = fnb.MutationConfig()
    m.node_add, m.conn_add, m.node_delete, m.conn_delete = 0.4, 0.6, 0.1, 0.1
    ev = Evolver(eng, NeatConfig(pop_size=500, compatibility_threshold=1.0, mutation=m), seed=3)
    ev.init_population()
    X, Y = regression_dataset(64, 3, 1, seed=1)
    for _ in range(30):
        ev.evaluate(X, Y)
        ev.step()
        assert ev.validate() == -1
    # a corrupted genome is reported with the reference's explanation
    n, c = ev.population()
    c[17, 0, 2] = 0.5 if not np.isnan(c[17, 0, 2]) else c[17, 0, 2]
    n[11, 0, 1] = np.nan
    ev.set_population(n, c)
    with pytest.raises(fnb.FlatneatError) as ei:
        ev.validate()
    assert ei.value.index == 11 and str(ei.value) == "corrupt_row: node row 0 partially NaN"
