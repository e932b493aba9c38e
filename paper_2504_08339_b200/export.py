"""Export of decoded genomes (SPEC.md:496-548 `export`): topology diagrams
(`to_dot`) and symbolic formulas (`to_formula`, `formula_tree`).

Host-only utilities for champions pulled off the device (SURVEY.md 8f item
4); they never run on the hot path.  Determinism: node statements by key,
edge statements by (in, out) key, one formula line per non-input node in the
reference's topological order (min key first, network.hpp:192-214), hidden
nodes named h0, h1, ... in that order, inputs i<k> and outputs o<k> by their
position in the input / output key lists.  Diagram numbers use 3 decimals
(SPEC.md:540); the FormulaTree keeps full FP64 values, so evaluating it
reproduces the forward pass (network.hpp:238-268) to rounding.
"""
from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .api import ACTIVATIONS, AGGREGATIONS, AttributeSchema, FlatneatError

_ACT_FN = {
    "identity": lambda x: x,
    "tanh": math.tanh,
    "sigmoid": lambda x: 1.0 / (1.0 + math.exp(-x)),
    "relu": lambda x: x if x > 0.0 else 0.0,
    "sin": math.sin,
}


@dataclass
class FormulaTree:
    """A node of the formula: an input leaf (`input_index` set) or an op with
    its activation, aggregation, bias, response and weighted children."""
    name: str
    input_index: Optional[int] = None
    act: str = "identity"
    agg: str = "sum"
    bias: float = 0.0
    resp: float = 1.0
    children: List[Tuple[float, "FormulaTree"]] = field(default_factory=list)

    def evaluate(self, inputs: Sequence[float], _memo: Optional[Dict[int, float]] = None) -> float:
        """FP64 value for `inputs`, with forward's semantics (network.hpp:252-264)."""
        memo = {} if _memo is None else _memo
        if id(self) in memo:
            return memo[id(self)]
        if self.input_index is not None:
            v = float(inputs[self.input_index])
        else:
            terms = [w * c.evaluate(inputs, memo) for w, c in self.children]
            if not terms:
                a = 1.0 if self.agg == "product" else 0.0
            elif self.agg in ("sum", "mean"):
                a = 0.0
                for t in terms:
                    a += t
                if self.agg == "mean":
                    a = a / len(terms)
            elif self.agg == "product":
                a = 1.0
                for t in terms:
                    a *= t
            else:  # max
                a = terms[0]
                for t in terms[1:]:
                    a = t if t > a else a
            v = _ACT_FN[self.act](self.resp * a + self.bias)
        memo[id(self)] = v
        return v


def _rows(nodes: np.ndarray, conns: np.ndarray):
    live_n = [r for r in range(nodes.shape[0]) if not np.isnan(nodes[r, 0])]
    live_c = [r for r in range(conns.shape[0]) if not np.isnan(conns[r, 0])]
    return live_n, live_c


def _topo_order(nodes, conns, live_n, live_c) -> List[int]:
    """Min-(key, row)-first Kahn order over enabled edges (network.hpp:192-214)."""
    row_of = {}
    for r in live_n:
        row_of.setdefault(int(nodes[r, 0]), r)
    indeg = {r: 0 for r in live_n}
    succ: Dict[int, List[int]] = {r: [] for r in live_n}
    for q in live_c:
        if conns[q, 2] != 1.0:
            continue
        a, b = row_of[int(conns[q, 0])], row_of[int(conns[q, 1])]
        indeg[b] += 1
        succ[a].append(b)
    heap = [(int(nodes[r, 0]), r) for r in live_n if indeg[r] == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        _, r = heapq.heappop(heap)
        order.append(r)
        for b in succ[r]:
            indeg[b] -= 1
            if indeg[b] == 0:
                heapq.heappush(heap, (int(nodes[b, 0]), b))
    if len(order) != len(live_n):
        raise FlatneatError(1 + 10, "cycle_detected: genome is not acyclic")  # Errc::cycle_detected
    return order


def _names(nodes, live_n, order, input_keys, output_keys) -> Dict[int, str]:
    names = {}
    for r in live_n:
        k = int(nodes[r, 0])
        if k in input_keys:
            names[r] = f"i{list(input_keys).index(k)}"
        elif k in output_keys:
            names[r] = f"o{list(output_keys).index(k)}"
    h = 0
    for r in order:
        if r not in names:
            names[r] = f"h{h}"
            h += 1
    return names


def to_dot(nodes, conns, input_keys: Sequence[int], output_keys: Sequence[int]) -> str:
    """Directed-graph text: inputs filled yellow, outputs
    doubled, hidden plain; disabled connections dashed; edge labels are the
    weights at 3 decimals; statements ordered by key."""
    nodes = np.asarray(nodes, dtype=np.float64)
    conns = np.asarray(conns, dtype=np.float64)
    live_n, live_c = _rows(nodes, conns)
    lines = ["digraph genome {", "  rankdir=LR;"]
    for r in sorted(live_n, key=lambda r: (int(nodes[r, 0]), r)):
        k = int(nodes[r, 0])
        if k in input_keys:
            style = 'shape=box, style=filled, fillcolor="yellow"'
        elif k in output_keys:
            style = "shape=doublecircle"
        else:
            style = "shape=circle"
        lines.append(f'  n{k} [label="{k}", {style}];')
    for q in sorted(live_c, key=lambda q: (int(conns[q, 0]), int(conns[q, 1]), q)):
        a, b, en, w = int(conns[q, 0]), int(conns[q, 1]), conns[q, 2], conns[q, 3]
        dashed = "" if en == 1.0 else ", style=dashed"
        lines.append(f'  n{a} -> n{b} [label="{w:.3f}"{dashed}];')
    lines.append("}")
    return "\n".join(lines) + "\n"


def formula_tree(nodes, conns, input_keys: Sequence[int], output_keys: Sequence[int],
                 schema: AttributeSchema = AttributeSchema()) -> Dict[str, FormulaTree]:
    """FormulaTree of every node by name."""
    nodes = np.asarray(nodes, dtype=np.float64)
    conns = np.asarray(conns, dtype=np.float64)
    live_n, live_c = _rows(nodes, conns)
    order = _topo_order(nodes, conns, live_n, live_c)
    names = _names(nodes, live_n, order, input_keys, output_keys)
    row_of = {}
    for r in live_n:
        row_of.setdefault(int(nodes[r, 0]), r)
    preds: Dict[int, List[Tuple[int, float]]] = {r: [] for r in live_n}
    for q in live_c:
        if conns[q, 2] == 1.0:
            preds[row_of[int(conns[q, 1])]].append((row_of[int(conns[q, 0])], float(conns[q, 3])))
    trees: Dict[int, FormulaTree] = {}
    for r in order:
        k = int(nodes[r, 0])
        if k in input_keys:
            trees[r] = FormulaTree(names[r], input_index=list(input_keys).index(k))
            continue
        t = FormulaTree(names[r], act=schema.activations[int(nodes[r, 4])],
                        agg=schema.aggregations[int(nodes[r, 3])], bias=float(nodes[r, 1]), resp=float(nodes[r, 2]))
        # edges in ascending source row, the forward's accumulation order (network.hpp:184-190)
        t.children = [(w, trees[src]) for src, w in sorted(preds[r], key=lambda e: e[0])]
        trees[r] = t
    return {trees[r].name: trees[r] for r in order}


def to_formula(nodes, conns, input_keys: Sequence[int], output_keys: Sequence[int],
               schema: AttributeSchema = AttributeSchema(), style: str = "plain") -> str:
    """One assignment per non-input node in topological order:
    `o0 = tanh(1.000 * (0.500 * i0 + -1.250 * h0) + 0.100)` in the plain
    style, math markup in the typeset style.  The response factor is shown
    only when it is not 1."""
    if style not in ("plain", "typeset"):
        raise ValueError("style must be 'plain' or 'typeset'")
    trees = formula_tree(nodes, conns, input_keys, output_keys, schema)
    tex = style == "typeset"

    def sym(name: str) -> str:
        return f"{name[0]}_{{{name[1:]}}}" if tex else name

    lines = []
    for name, t in trees.items():
        if t.input_index is not None:
            continue
        mul = r" \cdot " if tex else " * "
        terms = [f"{w:.3f}{mul}{sym(c.name)}" for w, c in t.children]
        if t.agg in ("sum", "mean"):
            inner = " + ".join(terms) if terms else "0.000"
            if t.agg == "mean" and terms:
                inner = (rf"\frac{{{inner}}}{{{len(terms)}}}" if tex else f"({inner}) / {len(terms)}")
        elif t.agg == "product":
            inner = (r" \cdot " if tex else " * ").join(f"({x})" for x in terms) if terms else "1.000"
        else:
            inner = ((r"\max(" if tex else "max(") + ", ".join(terms) + ")") if terms else "0.000"
        pre = inner if t.resp == 1.0 else f"{t.resp:.3f}{mul}({inner})"
        body = f"{pre} + {t.bias:.3f}"
        if t.act == "identity":
            rhs = (rf"\left({body}\right)" if tex else f"({body})")
        else:
            fn = {"tanh": r"\tanh", "sin": r"\sin"}.get(t.act, rf"\mathrm{{{t.act}}}") if tex else t.act
            rhs = (rf"{fn}\left({body}\right)" if tex else f"{fn}({body})")
        lines.append(f"{sym(name)} = {rhs}")
    return "\n".join(lines) + "\n"


__all__ = ["FormulaTree", "formula_tree", "to_dot", "to_formula", "ACTIVATIONS", "AGGREGATIONS"]
