"""CPU checks of the C4 HyperNEAT restatement (oracle/hyperneat.c) against an
independent numpy statement of the same rules."""
import numpy as np

import oracle_lib as ol
from paper_2504_08339_b200.synthetic import hyper_dynamics


def _np_rollout(cfg, W, A, B, s0):
    s = s0.copy()
    tot = 0.0
    for _ in range(cfg.steps):
        a = np.tanh(W[:, :-1] @ s + W[:, -1])
        s = A @ s + B @ a
        tot += -(s @ s) / cfg.n_obs - cfg.act_cost * (a @ a) / cfg.n_act
    return tot / cfg.steps


def test_queries_layout():
    cfg = ol.hyper_cfg()
    q = ol.hyper_queries(cfg)
    assert q.shape == (28 * 8, 5)
    # q = j * (n_obs + 1) + i: inputs along y = -1, outputs along y = +1, bias input last
    assert np.allclose(q[:28, 0], np.linspace(-1, 1, 28)) and np.all(q[:, 1] == -1) and np.all(q[:, 3] == 1)
    assert np.allclose(q[::28, 2], np.linspace(-1, 1, 8)) and np.all(q[:, 4] == 1)


def test_weight_rule():
    cfg = ol.hyper_cfg(threshold=0.2, max_weight=3.0)
    assert ol.hyper_weight(cfg, 0.19) == 0.0 and ol.hyper_weight(cfg, -0.1999) == 0.0
    assert ol.hyper_weight(cfg, 0.2) == 0.0
    assert ol.hyper_weight(cfg, 1.0) == 3.0 and ol.hyper_weight(cfg, 7.0) == 3.0 and ol.hyper_weight(cfg, -9.0) == -3.0
    assert abs(ol.hyper_weight(cfg, 0.6) - 1.5) < 1e-15 and abs(ol.hyper_weight(cfg, -0.6) + 1.5) < 1e-15


def test_rollout_matches_numpy():
    cfg = ol.hyper_cfg(steps=200)
    A, B, s0 = hyper_dynamics(seed=3)
    rng = np.random.default_rng(0)
    for _ in range(3):
        W = ol.hyper_substrate(cfg, rng.uniform(-1.2, 1.2, 28 * 8)).reshape(8, 28)
        got = ol.hyper_rollout(cfg, W, A, B, s0)
        want = _np_rollout(cfg, W, A, B, s0)
        assert abs(got - want) <= 1e-12 * abs(want), (got, want)


def test_dynamics_are_contracting():
    A, B, s0 = hyper_dynamics(seed=0)
    # closed-loop contraction: |A| + |B| max|W| < 1
    assert np.linalg.norm(A, 2) + np.linalg.norm(B, 2) * 3.0 * np.sqrt(8 * 28) < 0.951
    assert A.shape == (27, 27) and B.shape == (27, 8) and s0.shape == (27,)
    assert np.array_equal(A, A.astype(np.float32).astype(np.float64))
