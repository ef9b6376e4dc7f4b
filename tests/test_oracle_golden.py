"""Pin the CPU oracle (oracle/quadra_oracle.py) to the reference's own outputs.

The golden files were produced by running /root/reference's quadra.neurons
(oracle/gen_golden.py); the oracle must reproduce them to fp64 round-off.
"""
import numpy as np
import pytest

from conftest import golden_index, load_case
from oracle import quadra_oracle as Q

CASES = golden_index()["layers"]


def _params(z):
    return {k[2:]: v for k, v in z.items() if k.startswith("P_")}


@pytest.mark.parametrize("case", CASES, ids=[c["file"] for c in CASES])
def test_oracle_matches_reference_golden(case):
    z = load_case(case["file"])
    geo = Q.Geometry(case["kind"], case["k"], case["s"], case["p"])
    P = _params(z)
    y, a, b = Q.forward(case["family"], geo, P, z["x"])
    assert Q.rel_err(y, z["y"]) <= 1e-13
    if "a" in z:
        assert Q.rel_err(a, z["a"]) <= 1e-13 and Q.rel_err(b, z["b"]) <= 1e-13
    grads, dx = Q.symbolic_backward(case["family"], geo, P, z["x"], a, b, z["g"])
    assert Q.rel_err(dx, z["dx"]) <= 1e-13
    for role, g in grads.items():
        assert Q.rel_err(g, z["G_" + role]) <= 1e-13, role
    assert set(grads) == {k[2:] for k in z if k.startswith("G_")}


def test_known_answers():
    ka = golden_index()["known_answers"]
    # reference tests/test_neurons.py:117-132
    assert ka["y"] == 10.0 and ka["dx"] == 11.0
    P = {k: np.asarray(v, dtype=np.float64) for k, v in ka["scalar_params"].items()}
    geo = Q.Geometry("fc")
    y, a, b = Q.forward("proposed", geo, P, np.asarray([[2.0]]))
    assert y[0, 0] == 10.0
    _, dx = Q.symbolic_backward("proposed", geo, P, np.asarray([[2.0]]), a, b, np.asarray([[1.0]]))
    assert dx[0, 0] == 11.0


def test_zero_dy_gives_zero_gradients(rng):
    x, P, _ = Q.synthetic_layer("proposed", "conv", 2, 3, 4, 5, 5, 3, 1, 1, random_bias=True)
    geo = Q.Geometry("conv", 3, 1, 1)
    y, a, b = Q.forward("proposed", geo, P, x)
    grads, dx = Q.symbolic_backward("proposed", geo, P, x, a, b, np.zeros_like(y))
    assert (dx == 0).all() and all((g == 0).all() for g in grads.values())


def test_im2col_conv_matches_loops_exhaustive(rng):
    # reference tests/test_tensor.py:160-173 sweep, against the six-loop oracle
    for h in range(1, 9):
        for w in range(1, 9):
            for r in range(1, 4):
                for s in (1, 2):
                    for p in (0, 1):
                        if r > h + 2 * p or r > w + 2 * p:
                            continue
                        x = rng.normal(size=(2, 2, h, w))
                        k = rng.normal(size=(2, 2, r, r))
                        assert Q.rel_err(Q.conv_forward(x, k, s, p),
                                         Q.conv2d_loops(x, k, s, p)) <= 1e-12
