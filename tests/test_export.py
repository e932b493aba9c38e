"""Export module: to_dot / to_formula / FormulaTree.

The FormulaTree must reproduce the forward pass within 1e-9 (SPEC.md:505,
534) -- checked against the reference's own batch_forward (oracle/_ref) on
random valid genomes of the rich schema -- and every emitter must be
deterministic and follow the SPEC's examples."""
import numpy as np
import pytest

import oracle_lib as ol
from paper_2504_08339_b200.api import AttributeSchema
from paper_2504_08339_b200.export import formula_tree, to_dot, to_formula


def _identity_genome():
    n = np.full((4, 5), np.nan)
    n[0] = [0, 0.0, 1.0, 0, 0]   # input
    n[1] = [1, 0.0, 1.0, 0, 0]   # output, identity
    c = np.full((4, 4), np.nan)
    c[0] = [0, 1, 1.0, 1.0]
    return n, c


def test_spec_examples():
    n, c = _identity_genome()
    schema = AttributeSchema(["identity"], ["sum"])
    assert to_formula(n, c, [0], [1], schema) == "o0 = (1.000 * i0 + 0.000)\n"
    dot = to_dot(n, c, [0], [1])
    assert dot.count("->") == 1                       # exactly one edge statement
    assert to_dot(n, c, [0], [1]) == dot              # byte-identical
    # Fig. 5 shape: 3 inputs, 3 hidden, 1 output -> 7 node statements
    n7 = np.full((8, 5), np.nan)
    for r, k in enumerate([0, 1, 2, 3, 4, 5, 6]):
        n7[r] = [k, 0.1 * r, 1.0, 0, 0]
    c7 = np.full((12, 4), np.nan)
    edges = [(0, 4), (1, 4), (2, 5), (4, 6), (5, 6), (2, 3), (6, 3), (1, 5)]
    for q, (a, b) in enumerate(edges):
        c7[q] = [a, b, 1.0 if q != 2 else 0.0, 0.5 - 0.1 * q]
    d7 = to_dot(n7, c7, [0, 1, 2], [3])
    assert sum(1 for line in d7.splitlines() if "[label=" in line and "->" not in line) == 7
    assert d7.count("style=dashed") == 1
    f7 = to_formula(n7, c7, [0, 1, 2], [3], AttributeSchema(["tanh"], ["sum"]))
    assert [line.split(" = ")[0] for line in f7.splitlines()] == ["h0", "h1", "h2", "o0"]


def test_unused_hidden_node_still_emitted():
    n, c = _identity_genome()
    n[2] = [7, 0.3, 1.0, 0, 0]  # hidden, no edges
    f = to_formula(n, c, [0], [1], AttributeSchema(["identity"], ["sum"]))
    assert f.splitlines()[0] == "o0 = (1.000 * i0 + 0.000)"
    assert "h0 = (0.000 + 0.300)" in f


def test_cycle_is_rejected():
    n, c = _identity_genome()
    n[2] = [2, 0.0, 1.0, 0, 0]
    c[1] = [1, 2, 1.0, 1.0]
    c[2] = [2, 1, 1.0, 1.0]
    with pytest.raises(Exception, match="cycle_detected"):
        to_formula(n, c, [0], [1])


@pytest.mark.parametrize("seed", [1312, 90210])
def test_formula_tree_equals_forward(seed):
    schema = ol.RICH
    prob = ol.Problem(16, 60, [0, 1, 2], [3])
    nodes, conns = ol.random_genomes(seed, schema, 25, 16, 60)
    X = np.random.default_rng(seed).uniform(-2, 2, size=(100, 3))
    if ol.ref_available():
        st, bad, msg, want = ol.ref_batch_forward(prob, schema, nodes, conns, X)
        assert st == 0, msg
    else:
        want = np.stack([ol.oracle_forward(prob, schema, nodes[i], ol.oracle_transform(prob, schema, nodes[i],
                                                                                    conns[i]), X)
                         for i in range(nodes.shape[0])])
    sch = AttributeSchema(list(schema.activations), list(schema.aggregations))
    worst = 0.0
    for g in range(nodes.shape[0]):
        tree = formula_tree(nodes[g], conns[g], [0, 1, 2], [3], sch)
        for b in range(X.shape[0]):
            got = tree["o0"].evaluate(X[b])
            worst = max(worst, abs(got - want[g, b, 0]))
        for style in ("plain", "typeset"):
            text = to_formula(nodes[g], conns[g], [0, 1, 2], [3], sch, style)
            assert text == to_formula(nodes[g], conns[g], [0, 1, 2], [3], sch, style)
            assert text.count("\n") == sum(1 for k in nodes[g][:, 0] if not np.isnan(k) and k > 2)
    assert worst < 1e-9, worst
