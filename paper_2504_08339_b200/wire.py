"""Genome wire format: save_genome / load_genome (
SURVEY.md 8f item 3) -- host-side artifact plumbing for checkpoint/resume.

A self-describing structured text document: JSON with sorted keys, the
schema registries by name, the limits, and the dense NaN-padded row arrays
(genome.hpp:19-38) with `null` for NaN.  Floats are written with 17
significant digits, so output is byte-stable for identical genomes and
load(save(g)) restores every double bit for bit.  Errors follow the
reference's Errc vocabulary (errors.hpp:10-31): `parse_error` with
line/field context, `version_unsupported` for unknown versions.
"""
from __future__ import annotations

import json
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .api import FlatneatError

FORMAT = "flatneat-genome"
VERSION = 1
_PARSE_ERROR = 1 + 15          # Errc::parse_error
_VERSION_UNSUPPORTED = 1 + 16  # Errc::version_unsupported


def _num(x: float) -> str:
    if math.isnan(x):
        return "null"
    if math.isinf(x):
        raise FlatneatError(1 + 12, "non_finite_state: infinite value cannot be serialised")
    if x == int(x) and abs(x) < 2 ** 53:
        return str(int(x)) if not (x == 0 and math.copysign(1.0, x) < 0) else "-0.0"
    return "%.17g" % x


def _rows(a: np.ndarray) -> str:
    return "[" + ",".join("[" + ",".join(_num(float(v)) for v in row) + "]" for row in a) + "]"


def save_genome(nodes, conns, input_keys: Sequence[int], output_keys: Sequence[int],
                activations: Sequence[str] = ("tanh",), aggregations: Sequence[str] = ("sum",)) -> str:
    """One genome ([N_max,5] node rows, [C_max,4] connection rows) -> document text."""
    n = np.asarray(nodes, dtype=np.float64)
    c = np.asarray(conns, dtype=np.float64)
    if n.ndim != 2 or n.shape[1] != 5 or c.ndim != 2 or c.shape[1] != 4:
        raise FlatneatError(1 + 8, "shape_mismatch: genome rows must be [N,5] and [C,4]")
    # keys in sorted order (json.dumps(sort_keys=True) order), numbers formatted by hand
    parts = [
        '"activations":' + json.dumps(list(activations)),
        '"aggregations":' + json.dumps(list(aggregations)),
        '"conns":' + _rows(c),
        '"format":' + json.dumps(FORMAT),
        '"input_keys":' + json.dumps([int(k) for k in input_keys]),
        '"limits":{"max_conns":%d,"max_nodes":%d}' % (c.shape[0], n.shape[0]),
        '"nodes":' + _rows(n),
        '"output_keys":' + json.dumps([int(k) for k in output_keys]),
        '"version":%d' % VERSION,
    ]
    return "{" + ",".join(parts) + "}\n"


def _fail(msg: str, field: Optional[str] = None, line: Optional[int] = None):
    where = []
    if line is not None:
        where.append(f"line {line}")
    if field is not None:
        where.append(f"field '{field}'")
    raise FlatneatError(_PARSE_ERROR, "parse_error: " + msg + (" (" + ", ".join(where) + ")" if where else ""))


def _rows_in(doc: dict, field: str, width: int, count: int) -> np.ndarray:
    rows = doc.get(field)
    if not isinstance(rows, list) or len(rows) != count:
        _fail(f"expected {count} rows", field)
    out = np.empty((count, width))
    for i, row in enumerate(rows):
        if not isinstance(row, list) or len(row) != width:
            _fail(f"row {i} must have {width} entries", field)
        for j, v in enumerate(row):
            if v is None:
                out[i, j] = np.nan
            elif isinstance(v, (int, float)) and not isinstance(v, bool):
                out[i, j] = float(v)
            else:
                _fail(f"row {i} entry {j} is not a number or null", field)
    return out


def load_genome(text: str) -> Tuple[np.ndarray, np.ndarray, dict]:
    """Document text -> (nodes [N,5], conns [C,4], meta) ; meta holds the
    input/output keys and the schema registries by name."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        _fail(e.msg, line=e.lineno)
    if not isinstance(doc, dict):
        _fail("document is not an object")
    if doc.get("format") != FORMAT:
        _fail(f"format must be '{FORMAT}'", "format")
    version = doc.get("version")
    if not isinstance(version, int) or isinstance(version, bool):
        _fail("version must be an integer", "version")
    if version != VERSION:
        raise FlatneatError(_VERSION_UNSUPPORTED, f"version_unsupported: genome document version {version}")
    limits = doc.get("limits")
    if not isinstance(limits, dict):
        _fail("missing limits", "limits")
    N, C = limits.get("max_nodes"), limits.get("max_conns")
    if not all(isinstance(x, int) and not isinstance(x, bool) and x > 0 for x in (N, C)):
        _fail("limits must be positive integers", "limits")
    meta = {}
    for f in ("input_keys", "output_keys", "activations", "aggregations"):
        v = doc.get(f)
        want = int if f.endswith("keys") else str
        if not isinstance(v, list) or not all(isinstance(x, want) and not isinstance(x, bool) for x in v):
            _fail(f"must be a list of {want.__name__}", f)
        meta[f] = v
    return _rows_in(doc, "nodes", 5, N), _rows_in(doc, "conns", 4, C), meta


def save_population(pop_nodes, pop_conns, **kw) -> List[str]:
    """One document per genome of a PopulationTensors pair ([P,N,5], [P,C,4])."""
    return [save_genome(pop_nodes[i], pop_conns[i], **kw) for i in range(len(pop_nodes))]


def load_population(docs: Sequence[str]) -> Tuple[np.ndarray, np.ndarray, dict]:
    loaded = [load_genome(d) for d in docs]
    if not loaded:
        _fail("empty population")
    shapes = {(n.shape, c.shape) for n, c, _ in loaded}
    if len(shapes) != 1:
        raise FlatneatError(1 + 8, "shape_mismatch: genomes of a population must share limits")
    return np.stack([n for n, _, _ in loaded]), np.stack([c for _, c, _ in loaded]), loaded[0][2]


# ---- checkpoint / resume -------------------------------------
CHECKPOINT_FORMAT = "flatneat-b200-checkpoint"


def _fnum(x: float) -> str:
    if math.isinf(x):
        return '"inf"' if x > 0 else '"-inf"'
    return _num(x)


def save_checkpoint(state: dict, rep_nodes, rep_conns, pop_nodes, pop_conns, input_keys, output_keys,
                    activations=("tanh",), aggregations=("sum",)) -> str:
    """An evolver's run state (Evolver.get_state: seed, generation, innovation
    counter, species table with representatives) and its population as one
    document, in the genome format's conventions: sorted keys, 17 significant
    digits, null for the NaN padding -- load(save(x)) restores every bit."""
    rn = np.asarray(rep_nodes, dtype=np.float64)
    rc = np.asarray(rep_conns, dtype=np.float64)
    pn = np.asarray(pop_nodes, dtype=np.float64)
    pc = np.asarray(pop_conns, dtype=np.float64)
    k = len(state["species_id"])
    species = []
    for j in range(k):
        species.append("{" + ",".join([
            '"best":' + _fnum(float(state["species_best"][j])),
            '"id":%d' % state["species_id"][j],
            '"rep_conns":' + _rows(rc[j]),
            '"rep_nodes":' + _rows(rn[j]),
            '"size":%d' % state["species_size"][j],
            '"spawn":%d' % state["species_spawn"][j],
            '"stagnation":%d' % state["species_stagnation"][j],
        ]) + "}")
    parts = [
        '"activations":' + json.dumps(list(activations)),
        '"aggregations":' + json.dumps(list(aggregations)),
        '"format":' + json.dumps(CHECKPOINT_FORMAT),
        '"generation":%d' % state["generation"],
        '"input_keys":' + json.dumps([int(x) for x in input_keys]),
        '"limits":{"max_conns":%d,"max_nodes":%d}' % (pc.shape[1], pn.shape[1]),
        '"next_key":%d' % state["next_key"],
        '"next_species_id":%d' % state["next_species_id"],
        '"output_keys":' + json.dumps([int(x) for x in output_keys]),
        '"population":[' + ",".join('{"conns":%s,"nodes":%s}' % (_rows(pc[i]), _rows(pn[i]))
                                    for i in range(pn.shape[0])) + "]",
        '"seed":%d' % int(state["seed"]),
        '"species":[' + ",".join(species) + "]",
        '"version":%d' % VERSION,
    ]
    return "{" + ",".join(parts) + "}\n"


def load_checkpoint(text: str):
    """Document -> (state dict, rep_nodes [S,N,5], rep_conns [S,C,4],
    pop_nodes [P,N,5], pop_conns [P,C,4], meta)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        _fail(e.msg, line=e.lineno)
    if not isinstance(doc, dict) or doc.get("format") != CHECKPOINT_FORMAT:
        _fail(f"format must be '{CHECKPOINT_FORMAT}'", "format")
    version = doc.get("version")
    if not isinstance(version, int) or isinstance(version, bool):
        _fail("version must be an integer", "version")
    if version != VERSION:
        raise FlatneatError(_VERSION_UNSUPPORTED, f"version_unsupported: checkpoint document version {version}")

    def _int(f):
        v = doc.get(f)
        if not isinstance(v, int) or isinstance(v, bool):
            _fail("must be an integer", f)
        return v

    limits = doc.get("limits")
    if not isinstance(limits, dict):
        _fail("missing limits", "limits")
    N, Cm = limits.get("max_nodes"), limits.get("max_conns")
    if not all(isinstance(x, int) and not isinstance(x, bool) and x > 0 for x in (N, Cm)):
        _fail("limits must be positive integers", "limits")
    meta = {}
    for f in ("input_keys", "output_keys", "activations", "aggregations"):
        v = doc.get(f)
        want = int if f.endswith("keys") else str
        if not isinstance(v, list) or not all(isinstance(x, want) and not isinstance(x, bool) for x in v):
            _fail(f"must be a list of {want.__name__}", f)
        meta[f] = v
    pop = doc.get("population")
    if not isinstance(pop, list) or not pop:
        _fail("must be a non-empty list", "population")
    pn = np.stack([_rows_in(g, "nodes", 5, N) if isinstance(g, dict) else _fail("genome is not an object", "population")
                   for g in pop])
    pc = np.stack([_rows_in(g, "conns", 4, Cm) for g in pop])
    sp = doc.get("species")
    if not isinstance(sp, list) or len(sp) > 32:
        _fail("must be a list of at most 32 species", "species")
    state = dict(seed=_int("seed"), generation=_int("generation"), next_key=_int("next_key"),
                 next_species_id=_int("next_species_id"), species_id=[], species_best=[], species_stagnation=[],
                 species_size=[], species_spawn=[])
    rn = np.empty((len(sp), N, 5))
    rc = np.empty((len(sp), Cm, 4))
    for j, e in enumerate(sp):
        if not isinstance(e, dict):
            _fail(f"species {j} is not an object", "species")
        for f, key in (("id", "species_id"), ("stagnation", "species_stagnation"), ("size", "species_size"),
                       ("spawn", "species_spawn")):
            v = e.get(f)
            if not isinstance(v, int) or isinstance(v, bool):
                _fail(f"species {j} {f} must be an integer", "species")
            state[key].append(v)
        b = e.get("best")
        if b in ("inf", "-inf"):
            b = float(b)
        elif not isinstance(b, (int, float)) or isinstance(b, bool):
            _fail(f"species {j} best must be a number", "species")
        state["species_best"].append(float(b))
        rn[j] = _rows_in(e, "rep_nodes", 5, N)
        rc[j] = _rows_in(e, "rep_conns", 4, Cm)
    return state, rn, rc, pn, pc, meta
