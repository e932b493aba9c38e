"""Seeded synthetic populations and datasets of the BASELINE shapes.

Genomes are rank-ordered random DAGs with exact sizes: floor(fill*N_max)
nodes (inputs keys 0..I-1, outputs I..I+O-1, hidden after), floor(fill*C_max)
distinct rank-forward connections (15% disabled), weights and biases ~ N(0,1),
response 1.0 -- the same construction as the reference's test generator
(tests/support/generators.hpp:37-84) but with fixed counts so every genome
fills the configured limits.  Data generation only; nothing here is on the
timed path.
"""
from __future__ import annotations

import numpy as np


def synthetic_population(P: int, max_nodes: int, max_conns: int, fill: float = 0.75, num_inputs: int = 4,
                         num_outputs: int = 1, disabled_prob: float = 0.15, n_act: int = 1, n_agg: int = 1,
                         seed: int = 0, chunk: int = 4096):
    rng = np.random.default_rng(seed)
    n_nodes = max(num_inputs + num_outputs, int(fill * max_nodes))
    n_conns = int(fill * max_conns)
    I, O = num_inputs, num_outputs
    H = n_nodes - I - O
    # candidate (a, b) rank pairs with a < b and target not an input
    a_idx, b_idx = np.triu_indices(n_nodes, k=1)
    keep = b_idx >= I
    a_idx, b_idx = a_idx[keep], b_idx[keep]
    ncand = a_idx.size
    if n_conns > ncand:
        raise ValueError(f"{n_conns} connections exceed the {ncand} acyclic candidates")
    nodes = np.full((P, max_nodes, 5), np.nan)
    conns = np.full((P, max_conns, 4), np.nan)
    keys = np.arange(n_nodes, dtype=np.float64)
    for lo in range(0, P, chunk):
        hi = min(P, lo + chunk)
        n = hi - lo
        # rank position -> key: inputs, shuffled hidden, outputs
        hidden = I + O + np.argsort(rng.random((n, H)), axis=1)
        by_rank = np.concatenate([np.broadcast_to(np.arange(I), (n, I)), hidden,
                                  np.broadcast_to(np.arange(I, I + O), (n, O))], axis=1)
        nd = nodes[lo:hi]
        nd[:, :n_nodes, 0] = keys
        nd[:, :n_nodes, 1] = rng.standard_normal((n, n_nodes))
        nd[:, :n_nodes, 2] = 1.0
        nd[:, :n_nodes, 3] = rng.integers(0, n_agg, (n, n_nodes)) if n_agg > 1 else 0
        nd[:, :n_nodes, 4] = rng.integers(0, n_act, (n, n_nodes)) if n_act > 1 else 0
        pick = np.argpartition(rng.random((n, ncand)), n_conns - 1, axis=1)[:, :n_conns]
        pick.sort(axis=1)
        src = np.take_along_axis(by_rank, a_idx[pick], axis=1)
        dst = np.take_along_axis(by_rank, b_idx[pick], axis=1)
        cn = conns[lo:hi]
        cn[:, :n_conns, 0] = src
        cn[:, :n_conns, 1] = dst
        cn[:, :n_conns, 2] = (rng.random((n, n_conns)) >= disabled_prob).astype(np.float64)
        cn[:, :n_conns, 3] = rng.standard_normal((n, n_conns))
    return nodes, conns


def lineage_population(P: int, max_nodes: int, max_conns: int, ancestors: int = 10, fill: float = 0.75,
                       num_inputs: int = 4, num_outputs: int = 1, seed: int = 0):
    """A population descended from `ancestors` synthetic genomes, as a NEAT
    run's species are: genome i copies ancestor i % ancestors with mutation-like
    noise -- 80% of the connection weights and biases moved by N(0, 0.5^2),
    5% of the enabled connections disabled.  Markers (keys, endpoints) are
    the ancestor's, so a genome matches its own representative densely and
    the others as the ancestors overlap.  Returns (nodes, conns, anc_nodes,
    anc_conns)."""
    an, ac = synthetic_population(ancestors, max_nodes, max_conns, fill, num_inputs, num_outputs, seed=seed)
    rng = np.random.default_rng(seed + 1)
    idx = np.arange(P) % ancestors
    nodes, conns = an[idx].copy(), ac[idx].copy()
    live_c = ~np.isnan(conns[:, :, 0])
    live_n = ~np.isnan(nodes[:, :, 0])
    mw = live_c & (rng.random(live_c.shape) < 0.8)
    conns[:, :, 3] += np.where(mw, rng.normal(0.0, 0.5, live_c.shape), 0.0)
    off = live_c & (conns[:, :, 2] == 1.0) & (rng.random(live_c.shape) < 0.05)
    conns[:, :, 2] = np.where(off, 0.0, conns[:, :, 2])
    mb = live_n & (rng.random(live_n.shape) < 0.8)
    nodes[:, :, 1] += np.where(mb, rng.normal(0.0, 0.5, live_n.shape), 0.0)
    return nodes, conns, an, ac


def regression_dataset(batch: int, num_inputs: int = 4, num_outputs: int = 1, seed: int = 0):
    """X ~ U(-2, 2) sample-major [B, I]; y = a smooth fixed target [B, O]."""
    rng = np.random.default_rng(seed)
    X = rng.uniform(-2.0, 2.0, size=(batch, num_inputs))
    w = np.linspace(0.5, -0.5, num_inputs)
    base = np.sin(X @ w) + 0.25 * X[:, 0] * X[:, -1]
    Y = np.stack([np.tanh(base + 0.1 * o) for o in range(num_outputs)], axis=1)
    return X, Y


def xor_dataset(bias_input: bool = False):
    """XOR truth table; optional constant bias input."""
    X = np.array([[0, 0], [0, 1], [1, 0], [1, 1]], dtype=np.float64)
    if bias_input:
        X = np.concatenate([X, np.ones((4, 1))], axis=1)
    Y = np.array([[0], [1], [1], [0]], dtype=np.float64)
    return X, Y


def cppn_dataset(side: int = 256):
    """C3: CPPN queries over a side x side grid -- inputs
    (x, y, r = sqrt(x^2 + y^2), bias = 1) with x, y in [-1, 1] -- and a fixed
    target image (concentric rings) for the image-MSE fitness.  Returns
    (X [side^2, 4], Y [side^2, 1]) as float64."""
    t = np.linspace(-1.0, 1.0, side)
    yy, xx = np.meshgrid(t, t, indexing="ij")
    r = np.sqrt(xx * xx + yy * yy)
    X = np.stack([xx.ravel(), yy.ravel(), r.ravel(), np.ones(side * side)], axis=1)
    Y = (0.5 + 0.5 * np.cos(8.0 * np.pi * r)).reshape(-1, 1)
    return X, Y


def hyper_dynamics(num_obs: int = 27, num_act: int = 8, seed: int = 0, max_weight: float = 3.0):
    """C4: fixed seeded linear dynamics s' = A s + B a with
    |A|_2 = 0.85 and |B|_2 = 0.1 / (max_weight sqrt(num_act (num_obs + 1))), so
    the closed loop s -> A s + B tanh(W [s, 1]) is a contraction for every
    policy the substrate can express (|W|_2 <= |W|_F <= max_weight
    sqrt(num_act (num_obs + 1)), tanh is 1-Lipschitz): rollouts do not
    amplify rounding, and FP32 and FP64 rollouts stay within 1e-5 relative.
    s0 ~ U(-1, 1).  Values are rounded to float32 (the device computes in
    FP32) and returned as float64 A [num_obs, num_obs], B [num_obs, num_act],
    s0 [num_obs]."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((num_obs, num_obs))
    A *= 0.85 / np.linalg.norm(A, 2)
    B = rng.standard_normal((num_obs, num_act))
    B *= 0.1 / (max_weight * np.sqrt(num_act * (num_obs + 1))) / np.linalg.norm(B, 2)
    s0 = rng.uniform(-1.0, 1.0, num_obs)
    f = lambda x: x.astype(np.float32).astype(np.float64)
    return f(A), f(B), f(s0)


def cppn_population(P: int, max_nodes: int = 32, max_conns: int = 128, fill: float = 0.75, seed: int = 0):
    """C4 CPPNs: 5 inputs (x1, y1, x2, y2, bias) and 1 output; activation ids
    index the 5-function schema CPPN_ACTS."""
    return synthetic_population(P, max_nodes, max_conns, fill, num_inputs=5, num_outputs=1, n_act=5, seed=seed)


CPPN_ACTS = ["tanh", "sin", "sigmoid", "identity", "relu"]
