"""Genome save/load (paper_2504_08339_b200/wire.py):
lossless round trip, byte stability, and the parse_error /
version_unsupported contract."""
import json

import numpy as np
import pytest

from paper_2504_08339_b200.api import FlatneatError
from paper_2504_08339_b200.synthetic import synthetic_population
from paper_2504_08339_b200.wire import load_genome, load_population, save_genome, save_population

KW = dict(input_keys=[0, 1, 2, 3], output_keys=[4], activations=["tanh", "sigmoid"], aggregations=["sum"])


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.fixture(scope="module")
def pop():
    return synthetic_population(16, 24, 64, fill=0.75, seed=3)


def test_round_trip_bit_exact(pop):
    nodes, conns = pop
    for i in range(len(nodes)):
        text = save_genome(nodes[i], conns[i], **KW)
        n, c, meta = load_genome(text)
        np.testing.assert_array_equal(_bits(n), _bits(nodes[i]))  # NaN padding included
        np.testing.assert_array_equal(_bits(c), _bits(conns[i]))
        assert meta["input_keys"] == KW["input_keys"] and meta["activations"] == KW["activations"]


def test_awkward_values_round_trip(pop):
    nodes, conns = pop
    n, c = nodes[0].copy(), conns[0].copy()
    n[5, 1] = -0.0
    n[6, 1] = 5e-324          # smallest subnormal
    n[7, 1] = 1.0 / 3.0
    c[0, 3] = -1.7976931348623157e308
    c[1, 3] = 2.0 ** 60       # integral beyond 2^53
    n2, c2, _ = load_genome(save_genome(n, c, **KW))
    np.testing.assert_array_equal(_bits(n2), _bits(n))
    np.testing.assert_array_equal(_bits(c2), _bits(c))


def test_byte_stable_and_sorted(pop):
    nodes, conns = pop
    a = save_genome(nodes[1], conns[1], **KW)
    b = save_genome(nodes[1].copy(), conns[1].copy(), **KW)
    assert a == b
    doc = json.loads(a)
    assert list(doc) == sorted(doc)
    assert "null" in a  # NaN padding is the null literal


def test_population_round_trip(pop):
    nodes, conns = pop
    n, c, _ = load_population(save_population(nodes, conns, **KW))
    np.testing.assert_array_equal(_bits(n), _bits(nodes))
    np.testing.assert_array_equal(_bits(c), _bits(conns))


def test_truncated_document_is_parse_error(pop):
    text = save_genome(pop[0][0], pop[1][0], **KW)
    with pytest.raises(FlatneatError) as e:
        load_genome(text[: len(text) // 2])
    assert e.value.code == "parse_error" and "line" in str(e.value)


def test_unknown_version(pop):
    doc = json.loads(save_genome(pop[0][0], pop[1][0], **KW))
    doc["version"] = 99
    with pytest.raises(FlatneatError) as e:
        load_genome(json.dumps(doc))
    assert e.value.code == "version_unsupported"


@pytest.mark.parametrize("field,mutate", [
    ("nodes", lambda d: d["nodes"][0].pop()),
    ("conns", lambda d: d["conns"].pop()),
    ("nodes", lambda d: d["nodes"][1].__setitem__(1, "x")),
    ("limits", lambda d: d.__setitem__("limits", {"max_nodes": 0, "max_conns": 4})),
    ("input_keys", lambda d: d.__setitem__("input_keys", [0.5])),
])
def test_malformed_fields_name_the_field(pop, field, mutate):
    doc = json.loads(save_genome(pop[0][0], pop[1][0], **KW))
    mutate(doc)
    with pytest.raises(FlatneatError) as e:
        load_genome(json.dumps(doc))
    assert e.value.code == "parse_error" and field in str(e.value)


def test_infinite_value_is_refused(pop):
    n = pop[0][0].copy()
    n[5, 1] = np.inf
    with pytest.raises(FlatneatError) as e:
        save_genome(n, pop[1][0], **KW)
    assert e.value.code == "non_finite_state"


def test_checkpoint_document_round_trip():
    """save_checkpoint / load_checkpoint restore every double bit for bit,
    infinite best-ever values included, and reject other formats / versions."""
    import pytest
    from paper_2504_08339_b200.api import FlatneatError
    from paper_2504_08339_b200.wire import load_checkpoint, save_checkpoint
    rng = np.random.default_rng(0)
    P, N, Cm = 6, 10, 20
    pn = np.full((P, N, 5), np.nan)
    pc = np.full((P, Cm, 4), np.nan)
    pn[:, :4] = rng.normal(size=(P, 4, 5))
    pc[:, :7] = rng.normal(size=(P, 7, 4))
    rn, rc = pn[:2].copy(), pc[:2].copy()
    state = dict(seed=2**63 + 5, generation=12, next_key=345, next_species_id=7, species_id=[3, 6],
                 species_best=[float("-inf"), 0.1 + 0.2], species_stagnation=[4, 0], species_size=[4, 2],
                 species_spawn=[3, 3])
    text = save_checkpoint(state, rn, rc, pn, pc, [0, 1], [2], ["tanh"], ["sum"])
    st, a, b, n, c, meta = load_checkpoint(text)
    assert st == state
    for x, y in ((a, rn), (b, rc), (n, pn), (c, pc)):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
    assert meta == dict(input_keys=[0, 1], output_keys=[2], activations=["tanh"], aggregations=["sum"])
    assert save_checkpoint(st, a, b, n, c, [0, 1], [2], ["tanh"], ["sum"]) == text
    with pytest.raises(FlatneatError) as ei:
        load_checkpoint(text.replace('"version":1', '"version":2'))
    assert ei.value.code == "version_unsupported"
    with pytest.raises(FlatneatError) as ei:
        load_checkpoint(text.replace("flatneat-b200-checkpoint", "other"))
    assert ei.value.code == "parse_error"
