"""The drop-in boundary exercised from the REFERENCE side: the reference's own
Tape / backward sweep (tensor.py:134-185, :612-648) with its quadratic nodes
routed to the device through the plugin registry (tensor.py:598-609), as
INTEGRATION.md §"Python reference binding" describes.

The reference package is imported from ``baseline/_ref`` (the installed
reference, git-ignored, shipped with the snapshot) or, in the build container,
from /root/reference/pkg/src. It is test infrastructure here: the reference
computes the expected gradients on the CPU (fp64) and owns the tape.
"""
import importlib
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_REF_PATHS = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


def _import_reference():
    for p in _REF_PATHS:
        if os.path.isdir(os.path.join(p, "quadra")):
            if p not in sys.path:
                sys.path.insert(0, p)
            T = importlib.import_module("quadra.tensor")
            N = importlib.import_module("quadra.neurons")
            A = importlib.import_module("quadra.autobuild")
            return T, N, A
    pytest.skip("reference package not installed (baseline/_ref); run the pip install of DESIGN.md §0")


def _rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _case(A, T, N, family, kind, rng):
    k, s, p = (3, 2, 1) if kind == "conv" else (1, 1, 0)
    spec = A.QuadraticLayerSpec(kind=kind, family=family, in_dim=3, out_dim=4, kernel=k, stride=s, pad=p)
    params = {}
    for role, shape in N.param_shapes(spec).items():
        params[role] = T.Tensor(rng.normal(size=shape), is_param=True)
    xs = (2, 3, 7, 6) if kind == "conv" else (5, 3)
    x = rng.normal(size=xs)
    return spec, params, x


def _tape_grads(T, record, spec, params, x, r):
    """hybrid_tape_grads of the reference tests (test_neurons.py:160-170) with a
    pluggable record_symbolic."""
    xt = T.Tensor(x)
    tape = T.Tape(T.HYBRID)
    y = record(tape, spec, params, xt, tag="L")
    h = T.hadamard(y, T.Tensor(r), tape=tape)
    flat = T.reshape(h, (1, h.size), tape=tape)
    loss = T.rowsum(flat, tape=tape)
    wanted = [xt] + [params[k] for k in sorted(params)]
    grads = T.backward(tape, loss, params=wanted)
    return y.data, grads[xt.id].data, {k: grads[params[k].id].data for k in params}, tape


def test_registry_contract_cpu():
    """Without a GPU: the registry holds fn(node, g) rules for every reference
    family and install() swaps them into the reference registry and back."""
    from paper_2204_01701_b200 import neurons
    T, N, _ = _import_reference()
    for fam in N.QUADRATIC_FAMILIES:
        fn = neurons.SYMBOLIC_BACKWARD[fam]
        assert fn.__code__.co_argcount == 2 and fn.__code__.co_varnames[:2] == ("node", "g")
    before = dict(T.SYMBOLIC_BACKWARD)
    prev = neurons.install(T)
    try:
        for fam in N.QUADRATIC_FAMILIES:
            assert T.SYMBOLIC_BACKWARD[fam] is neurons._quad_node_backward
    finally:
        neurons.uninstall(T, prev)
    assert T.SYMBOLIC_BACKWARD == before


FAMS = [("proposed", "conv"), ("proposed", "fc"), ("t4", "conv"), ("t2", "conv"), ("t3", "conv"),
        ("t2and4", "conv"), ("t1_full", "fc")]


@pytest.mark.gpu
@pytest.mark.parametrize("family,kind", FAMS, ids=[f"{a}-{b}" for a, b in FAMS])
def test_reference_tape_through_device_backend(family, kind):
    """Our record_symbolic on the reference HYBRID tape, the reference sweep
    dispatching the node to the device rule: same loss gradients as the
    reference's own route (fp32 device arithmetic, 1e-4)."""
    from paper_2204_01701_b200 import neurons
    T, N, A = _import_reference()
    rng = np.random.default_rng(1234)
    if family.startswith("t1"):
        spec = A.QuadraticLayerSpec(kind="fc", family=family, in_dim=6, out_dim=1)
        params = {r: T.Tensor(rng.normal(size=sh), is_param=True) for r, sh in N.param_shapes(spec).items()}
        x = rng.normal(size=(5, 6))
    else:
        spec, params, x = _case(A, T, N, family, kind, rng)
    y0, _ = N.forward(spec, params, T.Tensor(x))
    r = rng.normal(size=y0.shape)
    y_ref, dx_ref, g_ref, tape_ref = _tape_grads(T, N.record_symbolic, spec, params, x, r)
    prev = neurons.install(T)
    try:
        y_dev, dx_dev, g_dev, tape_dev = _tape_grads(T, neurons.record_symbolic, spec, params, x, r)
    finally:
        neurons.uninstall(T, prev)
    assert _rel(y_dev, y_ref) <= 1e-4
    assert _rel(dx_dev, dx_ref) <= 1e-4, _rel(dx_dev, dx_ref)
    assert set(g_dev) == set(g_ref)
    for k in g_ref:
        assert _rel(g_dev[k], g_ref[k]) <= 1e-4, (k, _rel(g_dev[k], g_ref[k]))
    # the node retains the reference's minimal cache: identical HYBRID byte ledger
    assert tape_dev.layer_hybrid == tape_ref.layer_hybrid
    assert tape_dev.layer_auto == tape_ref.layer_auto


@pytest.mark.gpu
@pytest.mark.parametrize("family,kind", FAMS[:4], ids=[f"{a}-{b}" for a, b in FAMS[:4]])
def test_reference_recorded_node_device_backward(family, kind):
    """A node the REFERENCE recorded (its own CPU forward; arrays are fp64 host
    Tensors) swept with the device rule installed: the rule rebuilds the cache
    on the device from node.arrays."""
    from paper_2204_01701_b200 import neurons
    T, N, A = _import_reference()
    rng = np.random.default_rng(77)
    spec, params, x = _case(A, T, N, family, kind, rng)
    y0, _ = N.forward(spec, params, T.Tensor(x))
    r = rng.normal(size=y0.shape)
    _, dx_ref, g_ref, _ = _tape_grads(T, N.record_symbolic, spec, params, x, r)
    prev = neurons.install(T)
    try:
        _, dx_dev, g_dev, _ = _tape_grads(T, N.record_symbolic, spec, params, x, r)
    finally:
        neurons.uninstall(T, prev)
    assert _rel(dx_dev, dx_ref) <= 1e-4
    for k in g_ref:
        assert _rel(g_dev[k], g_ref[k]) <= 1e-4, k


def test_init_params_same_draws_as_reference():
    """neurons.init_params consumes the same Generator draws, in the same role
    order, as the reference init_params (neurons.py:132-147): identical values
    (our fp32 masters = the reference's fp64 draws rounded) and the same
    generator state afterwards, for every family and kind."""
    import torch
    from paper_2204_01701_b200 import neurons
    from paper_2204_01701_b200.spec import QuadraticLayerSpec
    T, N, A = _import_reference()
    cases = []
    for fam in N.FAMILIES:
        if fam.startswith("t1"):
            cases.append(("fc", fam, 7, 1, 1))
            continue
        cases += [("fc", fam, 6, 5, 1), ("conv", fam, 3, 4, 3), ("dwconv", fam, 4, 4, 3)]
    for kind, fam, c, f, k in cases:
        rspec = A.QuadraticLayerSpec(kind=kind, family=fam, in_dim=c, out_dim=f, kernel=k, stride=1,
                                     pad=k // 2)
        ospec = QuadraticLayerSpec(kind=kind, family=fam, in_dim=c, out_dim=f, kernel=k, stride=1, pad=k // 2)
        r1, r2 = np.random.default_rng(99), np.random.default_rng(99)
        ref = N.init_params(rspec, r1)
        ours = neurons.init_params(ospec, r2, device="cpu")
        assert list(ref) == list(ours), (kind, fam)
        for role in ref:
            assert torch.equal(ours[role], torch.as_tensor(ref[role].data, dtype=torch.float32)), (kind, fam, role)
        assert r1.integers(1 << 62) == r2.integers(1 << 62), (kind, fam)
