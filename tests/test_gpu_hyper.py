"""GPU parity for BASELINE config 4 (HyperNEAT, csrc/hyper.cu) through the C ABI.

Checker: the CPPN outputs come from the reference's own batch_forward
(oracle/_ref) in FP64; substrate weights and the rollout from the FP64
restatement oracle/hyperneat.c (the reference has no HyperNEAT code, so the
substrate / rollout rules are "parity unpinned" -- DESIGN.md section 9).
Bars: weights within the FP32 forward's tolerance wherever the CPPN output is
not within 1e-4 of the threshold (a FP32 / FP64 difference there may flip a
weight to zero); fitness within 1e-5 relative."""
import numpy as np
import pytest

import oracle_lib as ol

pytestmark = pytest.mark.gpu

RTOL = 1e-5


@pytest.fixture(scope="module")
def fnb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_08339_b200 as m
    return m


def _setup(fnb, P, seed, steps=1000, limits=(32, 128)):
    from paper_2504_08339_b200.synthetic import CPPN_ACTS, cppn_population, hyper_dynamics
    nodes, conns = cppn_population(P, *limits, seed=seed)
    A, B, s0 = hyper_dynamics(seed=seed)
    schema = ol.SchemaSpec(CPPN_ACTS, ["sum"])
    prob = ol.Problem(limits[0], limits[1], [0, 1, 2, 3, 4], [5])
    eng = fnb.Engine(fnb.GenomeLimits(*limits), [0, 1, 2, 3, 4], [5], fnb.AttributeSchema(CPPN_ACTS, ["sum"]))
    cfg = fnb.HyperConfig(steps=steps)
    ocfg = ol.hyper_cfg(steps=steps)
    return nodes, conns, A, B, s0, schema, prob, eng, cfg, ocfg


@pytest.mark.parametrize("seed", [0, 9])
def test_substrate_weights_and_fitness(fnb, seed):
    nodes, conns, A, B, s0, schema, prob, eng, cfg, ocfg = _setup(fnb, 96, seed)
    fit, W = eng.hyper_evaluate(nodes, conns, cfg, A, B, s0, weights=True)
    y = ol.hyper_cppn_outputs(prob, schema, nodes, conns, ocfg)          # FP64 reference CPPNs
    clean = 0
    for p in range(nodes.shape[0]):
        Wr = ol.hyper_substrate(ocfg, y[p]).reshape(8, 28)
        near = np.abs(np.abs(np.clip(y[p], -1, 1)) - 0.2).reshape(8, 28) < 1e-4
        np.testing.assert_allclose(W[p][~near], Wr[~near], rtol=1e-5, atol=3e-5)
        # the rollout on the device's own weights: isolates the FP32 dynamics
        f_own = ol.hyper_rollout(ocfg, W[p].astype(np.float64), A, B, s0)
        assert abs(fit[p] - f_own) <= RTOL * abs(f_own), (p, fit[p], f_own)
        if not near.any():  # end to end against the FP64 pipeline
            f_ref = ol.hyper_rollout(ocfg, Wr, A, B, s0)
            assert abs(fit[p] - f_ref) <= RTOL * abs(f_ref) + 1e-9, (p, fit[p], f_ref)
            clean += 1
    assert clean > 50


def test_device_layer_equals_host_layer(fnb):
    import torch
    nodes, conns, A, B, s0, schema, prob, eng, cfg, ocfg = _setup(fnb, 40, 5, steps=300)
    fit = eng.hyper_evaluate(nodes, conns, cfg, A, B, s0)
    dev = torch.device("cuda", 0)
    dn, dc = torch.from_numpy(nodes).to(dev), torch.from_numpy(conns).to(dev)
    nets = eng.alloc_nets(40)
    st = torch.cuda.current_stream()
    eng.transform_d(dn, dc, nets, st)
    f = lambda x: torch.from_numpy(x.astype(np.float32)).to(dev)
    out = torch.empty(40, dtype=torch.float64, device=dev)
    eng.hyper_evaluate_d(nets, 40, cfg, f(A), f(B), f(s0), out, stream=st)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), fit)


def test_errors(fnb):
    nodes, conns, A, B, s0, schema, prob, eng, cfg, ocfg = _setup(fnb, 4, 1, steps=10)
    bad = fnb.HyperConfig(num_obs=40, steps=10)
    with pytest.raises(fnb.FlatneatError) as ei:
        eng.hyper_evaluate(nodes, conns, bad, np.zeros((40, 40)), np.zeros((40, 8)), np.zeros(40))
    assert ei.value.code == "config_error"
    e4 = fnb.Engine(fnb.GenomeLimits(32, 128), [0, 1, 2, 3], [4], fnb.AttributeSchema())
    with pytest.raises(fnb.FlatneatError) as ei:
        e4.hyper_evaluate(nodes, conns, cfg, A, B, s0)
    assert ei.value.code == "shape_mismatch"
    # a cyclic CPPN is reported like every transform error (lowest genome)
    c2 = conns.copy()
    c2[2, 0] = [5, 5, 1.0, 0.5]
    with pytest.raises(fnb.FlatneatError) as ei:
        eng.hyper_evaluate(nodes, c2, cfg, A, B, s0)
    assert ei.value.index == 2 and ei.value.code == "cycle_detected"
