"""GPU parity: the CUDA kernels (through the C ABI) vs the CPU oracle.

Tolerances (BASELINE.json north_star): rel_err (reference tests/oracles.py:98-102)
<= 1e-4 for fp32, <= 2e-2 for bf16; the oracle consumes the SAME cast input
values upcast to fp64, so the comparison measures kernel error only.
"""
import numpy as np
import pytest
import torch

from conftest import golden_index, load_case
from oracle import quadra_oracle as Q

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


def _spec(family, kind, c, f, k=1, s=1, p=0):
    from paper_2204_01701_b200.spec import QuadraticLayerSpec
    return QuadraticLayerSpec(kind=kind, family=family, in_dim=c, out_dim=f, kernel=k, stride=s,
                              pad=p)


def _q(a, dtype):
    """Round an fp64 array to the run dtype and back (what the kernel sees)."""
    return torch.as_tensor(a).to(dtype).to(torch.float64).numpy()


def run_device(family, kind, x, P, g, dtype, k=1, s=1, p=0, flags=0):
    from paper_2204_01701_b200 import neurons
    c = x.shape[1]
    f = g.shape[1]
    spec = _spec(family, kind, c, f, k, s, p)
    dev = torch.device("cuda")
    xt = torch.as_tensor(x, device=dev).to(dtype)
    params = {r: torch.as_tensor(v, dtype=torch.float32, device=dev) for r, v in P.items()}
    y, cache = neurons.forward(spec, params, xt, dtype=dtype, flags=flags)
    grads, dx = neurons.symbolic_backward(spec, params, cache, torch.as_tensor(g, device=dev).to(dtype))
    torch.cuda.synchronize()
    cv = lambda t: None if t is None else t.detach().to(torch.float64).cpu().numpy()  # noqa: E731
    return (cv(y), cv(cache.a), cv(cache.b), {r: cv(v) for r, v in grads.items()}, cv(dx),
            neurons.device_path(spec, x.shape, dtype, flags))


def check_against_oracle(family, kind, x, P, g, dtype, k=1, s=1, p=0, flags=0, tol=None):
    """Run device + oracle on identical (dtype-rounded) inputs; assert parity."""
    tol = tol or TOL[dtype]
    xq = _q(x, dtype)
    gq = _q(g, dtype)
    # weights are fp32 masters, cast to the compute dtype by the packer
    Pq = {r: (_q(v, dtype) if not r.startswith("b") else _q(v, torch.float32)) for r, v in P.items()}
    y, a, b, grads, dx, path = run_device(family, kind, xq, P, gq, dtype, k, s, p, flags)
    geo = Q.Geometry(kind, k, s, p)
    ry, ra, rb = Q.forward(family, geo, Pq, xq)
    assert Q.rel_err(y, ry) <= tol, ("y", Q.rel_err(y, ry))
    if ra is not None:
        assert Q.rel_err(a, ra) <= tol and Q.rel_err(b, rb) <= tol
    # oracle backward uses the kernel's own (rounded) a, b cache like the reference
    ca = a if a is not None else None
    cb = b if b is not None else None
    rg, rdx = Q.symbolic_backward(family, geo, Pq, xq, ca, cb, gq)
    assert Q.rel_err(dx, rdx) <= tol, ("dx", Q.rel_err(dx, rdx))
    assert set(grads) == set(rg)
    for role in rg:
        assert Q.rel_err(grads[role], rg[role]) <= tol, (role, Q.rel_err(grads[role], rg[role]))
    return path


GOLD = golden_index()["layers"]


@pytest.mark.parametrize("case", GOLD, ids=[c["file"] for c in GOLD])
def test_golden_cases_fp32(case):
    """Every reference golden case (incl. k3/s2/p1 and k2/s1/p0) in fp32 against
    the REFERENCE's own outputs."""
    z = load_case(case["file"])
    P = {k[2:]: v for k, v in z.items() if k.startswith("P_")}
    y, a, b, grads, dx, _ = run_device(case["family"], case["kind"], z["x"], P, z["g"],
                                       torch.float32, case["k"], case["s"], case["p"])
    assert Q.rel_err(y, z["y"]) <= 1e-4
    assert Q.rel_err(dx, z["dx"]) <= 1e-4
    for role in grads:
        assert Q.rel_err(grads[role], z["G_" + role]) <= 1e-4, role


@pytest.mark.parametrize("case", GOLD, ids=[c["file"] for c in GOLD])
def test_golden_cases_bf16(case):
    z = load_case(case["file"])
    P = {k[2:]: v for k, v in z.items() if k.startswith("P_")}
    check_against_oracle(case["family"], case["kind"], z["x"], P, z["g"], torch.bfloat16,
                         case["k"], case["s"], case["p"])


# shapes that tile onto the tcgen05 kernels (C, F multiples of 64, stride 1)
TC_CASES = [
    # family, kind, n, c, f, h, w, k, s, p
    ("proposed", "conv", 2, 64, 64, 8, 8, 3, 1, 1),
    ("proposed", "conv", 3, 64, 128, 10, 12, 3, 1, 1),
    ("proposed", "conv", 2, 128, 64, 6, 6, 1, 1, 0),
    ("proposed", "conv", 2, 64, 64, 9, 7, 2, 1, 0),
    ("proposed", "conv", 8, 64, 64, 32, 32, 3, 1, 1),       # BASELINE C2 geometry, batch 8
    ("proposed", "conv", 4, 256, 256, 7, 7, 3, 1, 1),       # C5 512@7-like, dgrad N=256
    ("t4", "conv", 2, 64, 64, 8, 8, 3, 1, 1),
    ("t4", "conv", 2, 64, 128, 11, 9, 3, 1, 1),
    ("t2", "conv", 2, 64, 64, 8, 8, 3, 1, 1),
    ("t2_linear", "conv", 2, 64, 64, 8, 8, 3, 1, 1),
    ("t2_linear", "conv", 2, 128, 64, 5, 6, 3, 1, 1),
    ("first_order", "conv", 2, 64, 128, 8, 8, 3, 1, 1),
    # CTA-pair / halo kernel (conv2): odd batch, streamed B, dual-K, k2/k5
    ("proposed", "conv", 3, 64, 64, 16, 16, 3, 1, 1),
    ("proposed", "conv", 2, 128, 128, 14, 20, 3, 1, 1),
    ("t4", "conv", 4, 64, 64, 16, 16, 3, 1, 1),
    ("t2", "conv", 2, 64, 64, 16, 16, 3, 1, 1),
    ("t2_linear", "conv", 2, 64, 64, 16, 16, 3, 1, 1),
    ("first_order", "conv", 2, 64, 128, 16, 16, 3, 1, 1),
    ("proposed", "conv", 2, 64, 64, 13, 17, 2, 1, 0),
    ("proposed", "conv", 2, 64, 64, 12, 12, 5, 1, 2),
    # stride 2 (ResNet downsampling) on its own output grid: traversal-stride-2
    # x maps for the fprop / wgrad, four output-parity classes for the dgrad
    # (odd H / W: classes of unequal size; k2 p0 / k5 p2: other tap parities);
    # t2_linear keeps the stride-1 grid + subsampled epilogue / upsampled operand
    ("proposed", "conv", 2, 64, 128, 28, 28, 3, 2, 1),
    ("proposed", "conv", 3, 64, 64, 29, 27, 3, 2, 1),
    ("proposed", "conv", 4, 128, 256, 14, 14, 3, 2, 1),
    ("proposed", "conv", 2, 64, 64, 15, 13, 2, 2, 0),
    ("proposed", "conv", 3, 64, 64, 11, 10, 5, 2, 2),
    ("t4", "conv", 2, 64, 64, 16, 16, 3, 2, 1),
    ("t4", "conv", 5, 128, 64, 8, 8, 3, 2, 1),
    ("first_order", "conv", 2, 64, 128, 16, 16, 3, 2, 1),
    ("t2_linear", "conv", 2, 64, 64, 16, 18, 3, 2, 1),
    # 1x1 stride 2 (ResNet shortcuts): three of the four parity classes get no tap
    ("first_order", "conv", 2, 64, 128, 16, 16, 1, 2, 0),
    ("proposed", "conv", 3, 64, 64, 9, 11, 1, 2, 0),
    ("proposed", "fc", 200, 128, 192, 1, 1, 1, 1, 0),
    ("t4", "fc", 130, 64, 64, 1, 1, 1, 1, 0),
    ("t2_linear", "fc", 64, 128, 64, 1, 1, 1, 1, 0),
    # t3 (a recomputed in the backward) and t2and4 (dual K with structural zeros)
    ("t3", "conv", 2, 64, 64, 8, 8, 3, 1, 1),
    ("t3", "conv", 2, 64, 128, 16, 16, 3, 1, 1),
    ("t3", "fc", 96, 128, 64, 1, 1, 1, 1, 0),
    ("t2and4", "conv", 2, 64, 64, 8, 8, 3, 1, 1),
    ("t2and4", "conv", 2, 64, 64, 16, 16, 3, 1, 1),
    ("t2and4", "conv", 2, 64, 64, 16, 18, 3, 2, 1),
    ("t2and4", "fc", 64, 64, 128, 1, 1, 1, 1, 0),
]


@pytest.mark.parametrize("case", TC_CASES, ids=[f"{c[0]}-{c[1]}-{c[3]}x{c[4]}-{c[5]}x{c[6]}-k{c[7]}p{c[9]}"
                                               for c in TC_CASES])
def test_tcgen05_path_parity(case):
    fam, kind, n, c, f, h, w, k, s, p = case
    x, P, g = Q.synthetic_layer(fam, kind, n, c, f, h, w, k, s, p, seed=7, random_bias=True)
    path = check_against_oracle(fam, kind, x, P, g, torch.bfloat16, k, s, p)
    assert path == 1, "expected the tcgen05 kernels for this shape"


@pytest.mark.parametrize("case", TC_CASES[:4] + TC_CASES[8:10], ids=str)
def test_tcgen05_matches_cuda_core_path(case):
    """Same bf16 inputs through the tcgen05 kernels and the CUDA-core kernels."""
    from paper_2204_01701_b200 import _lib
    fam, kind, n, c, f, h, w, k, s, p = case
    x, P, g = Q.synthetic_layer(fam, kind, n, c, f, h, w, k, s, p, seed=11, random_bias=True)
    xq, gq = _q(x, torch.bfloat16), _q(g, torch.bfloat16)
    r1 = run_device(fam, kind, xq, P, gq, torch.bfloat16, k, s, p)
    r0 = run_device(fam, kind, xq, P, gq, torch.bfloat16, k, s, p, flags=_lib.FLAG_FORCE_SIMT)
    assert r1[5] == 1 and r0[5] == 0
    assert Q.rel_err(r1[0], r0[0]) <= 1e-2
    assert Q.rel_err(r1[4], r0[4]) <= 1e-2
    for role in r1[3]:
        assert Q.rel_err(r1[3][role], r0[3][role]) <= 1e-2, role


@pytest.mark.parametrize("case", [c for c in TC_CASES if c[1] == "conv" and c[5] >= 12], ids=str)
def test_pair_halo_kernel_matches_v1(case):
    """conv2 (CTA pairs, halo reuse) vs the v1 tcgen05 kernels on identical inputs."""
    from paper_2204_01701_b200 import _lib
    fam, kind, n, c, f, h, w, k, s, p = case
    x, P, g = Q.synthetic_layer(fam, kind, n, c, f, h, w, k, s, p, seed=13, random_bias=True)
    xq, gq = _q(x, torch.bfloat16), _q(g, torch.bfloat16)
    r2 = run_device(fam, kind, xq, P, gq, torch.bfloat16, k, s, p)
    r1 = run_device(fam, kind, xq, P, gq, torch.bfloat16, k, s, p, flags=_lib.FLAG_TC_V1)
    for i in (0, 4):
        assert Q.rel_err(r2[i], r1[i]) <= 1e-2, i
    for role in r1[3]:
        assert Q.rel_err(r2[3][role], r1[3][role]) <= 1e-2, role


# small output grids on the v1 kernels: the K loop is split across CTAs into fp32
# partials that splitk_finish folds and runs the epilogue on
SPLITK_CASES = [
    ("proposed", "conv", 2, 128, 128, 4, 4, 3, 1, 1),
    ("proposed", "conv", 4, 256, 256, 2, 2, 3, 1, 1),
    ("t4", "conv", 2, 128, 64, 4, 4, 3, 1, 1),
    ("t2", "conv", 2, 128, 128, 4, 4, 3, 1, 1),
    ("t2_linear", "conv", 2, 128, 64, 4, 4, 3, 1, 1),
    ("first_order", "conv", 2, 256, 256, 3, 3, 3, 1, 1),
    ("proposed", "fc", 64, 1024, 256, 1, 1, 1, 1, 0),
    ("proposed", "conv", 2, 512, 512, 3, 3, 3, 1, 1),  # + the tiled weight pack (large layer)
]


def _kernel_names(fn):
    from paper_2204_01701_b200 import _lib
    lib = _lib.load()
    torch.cuda.synchronize()
    lib.qd_profile(1)
    try:
        out = fn()
        torch.cuda.synchronize()
        names = [n for n, _ in _lib.profile_read()]
    finally:
        lib.qd_profile(0)
    return out, names


@pytest.mark.parametrize("case", SPLITK_CASES, ids=str)
def test_splitk_v1_parity(case, monkeypatch):
    fam, kind, n, c, f, h, w, k, s, p = case
    x, P, g = Q.synthetic_layer(fam, kind, n, c, f, h, w, k, s, p, seed=17, random_bias=True)
    xq, gq = _q(x, torch.bfloat16), _q(g, torch.bfloat16)
    path, names = _kernel_names(lambda: check_against_oracle(fam, kind, x, P, g, torch.bfloat16, k, s, p))
    assert path == 1
    assert "splitk_finish" in names, names
    r_split = run_device(fam, kind, xq, P, gq, torch.bfloat16, k, s, p)
    monkeypatch.setenv("QD_NO_SPLITK", "1")
    r_whole, names1 = _kernel_names(lambda: run_device(fam, kind, xq, P, gq, torch.bfloat16, k, s, p))
    assert "splitk_finish" not in names1
    for i in (0, 4):
        assert Q.rel_err(r_split[i], r_whole[i]) <= 1e-2, i
    for role in r_whole[3]:
        assert Q.rel_err(r_split[3][role], r_whole[3][role]) <= 1e-2, role


def test_c1_fc_fp32():
    """BASELINE config 1: fc 256x512->512, fp32, Kaiming-uniform, b=0."""
    x, P, g = Q.synthetic_layer("proposed", "fc", 256, 512, 512, seed=0)
    check_against_oracle("proposed", "fc", x, P, g, torch.float32)


# fp32 on the tensor cores (path 3): split bf16 operands, 3 products per GEMM, 1e-4
X3_CASES = [
    # family, kind, n, c, f, h, w, k, s, p
    ("proposed", "conv", 2, 64, 64, 8, 8, 3, 1, 1),
    ("proposed", "conv", 3, 64, 128, 10, 12, 3, 1, 1),
    ("proposed", "conv", 2, 128, 64, 6, 6, 1, 1, 0),
    ("proposed", "conv", 2, 64, 64, 9, 7, 2, 1, 0),
    ("t4", "conv", 2, 64, 128, 11, 9, 3, 1, 1),
    ("first_order", "conv", 2, 64, 128, 8, 8, 3, 1, 1),
    ("proposed", "conv", 2, 256, 256, 4, 4, 3, 1, 1),  # split K (small grid)
    ("proposed", "fc", 200, 128, 192, 1, 1, 1, 1, 0),
    ("t4", "fc", 130, 64, 64, 1, 1, 1, 1, 0),
    ("first_order", "fc", 64, 256, 128, 1, 1, 1, 1, 0),
]


@pytest.mark.parametrize("case", X3_CASES, ids=[f"{c[0]}-{c[1]}-{c[3]}x{c[4]}-{c[5]}x{c[6]}-k{c[7]}"
                                               for c in X3_CASES])
def test_fp32_tensor_core_path_parity(case):
    fam, kind, n, c, f, h, w, k, s, p = case
    x, P, g = Q.synthetic_layer(fam, kind, n, c, f, h, w, k, s, p, seed=21, random_bias=True)
    path = check_against_oracle(fam, kind, x, P, g, torch.float32, k, s, p)
    assert path == 3, "expected the fp32 split tensor-core path for this shape"


@pytest.mark.parametrize("case", X3_CASES[:3] + X3_CASES[7:8], ids=str)
def test_fp32_tensor_core_matches_ffma_path(case):
    """fp32 through the split tensor-core kernels and the exact FFMA kernels."""
    from paper_2204_01701_b200 import _lib
    fam, kind, n, c, f, h, w, k, s, p = case
    x, P, g = Q.synthetic_layer(fam, kind, n, c, f, h, w, k, s, p, seed=23, random_bias=True)
    r3 = run_device(fam, kind, x, P, g, torch.float32, k, s, p)
    r0 = run_device(fam, kind, x, P, g, torch.float32, k, s, p, flags=_lib.FLAG_FORCE_SIMT)
    assert r3[5] == 3 and r0[5] == 0
    for i in (0, 4):
        assert Q.rel_err(r3[i], r0[i]) <= 1e-4, i
    for role in r3[3]:
        assert Q.rel_err(r3[3][role], r0[3][role]) <= 1e-4, role


def test_variants_fp32_conv():
    for fam in ("proposed", "t4", "t2", "t2_linear", "first_order"):
        x, P, g = Q.synthetic_layer(fam, "conv", 2, 5, 6, 7, 6, 3, 2, 1, seed=3, random_bias=True)
        check_against_oracle(fam, "conv", x, P, g, torch.float32, 3, 2, 1)


def test_c2_full_batch_properties():
    """BASELINE config 2 at full size (128x64x32x32 -> 64, bf16): per-sample
    outputs vs the oracle on a slice, and batch-linearity of dW/db."""
    from paper_2204_01701_b200 import neurons
    fam, n = "proposed", 128
    x, P, g = Q.synthetic_layer(fam, "conv", n, 64, 64, 32, 32, 3, 1, 1, seed=0)
    dt = torch.bfloat16
    xq, gq = _q(x, dt), _q(g, dt)
    y, a, b, grads, dx, path = run_device(fam, "conv", xq, P, gq, dt, 3, 1, 1)
    assert path == 1
    assert np.isfinite(y).all() and np.isfinite(dx).all()
    geo = Q.Geometry("conv", 3, 1, 1)
    Pq = {r: (_q(v, dt) if not r.startswith("b") else v) for r, v in P.items()}
    sl = slice(0, 4)
    ry, ra, rb = Q.forward(fam, geo, Pq, xq[sl])
    assert Q.rel_err(y[sl], ry) <= 2e-2
    _, rdx = Q.symbolic_backward(fam, geo, Pq, xq[sl], a[sl], b[sl], gq[sl])
    assert Q.rel_err(dx[sl], rdx) <= 2e-2
    h = n // 2
    _, _, _, g1, _, _ = run_device(fam, "conv", xq[:h], P, gq[:h], dt, 3, 1, 1)
    _, _, _, g2, _, _ = run_device(fam, "conv", xq[h:], P, gq[h:], dt, 3, 1, 1)
    for role in grads:
        assert Q.rel_err(grads[role], g1[role] + g2[role]) <= 1e-2, role


def test_deterministic_replay():
    """Bitwise-identical outputs and gradients on replay."""
    x, P, g = Q.synthetic_layer("proposed", "conv", 4, 64, 64, 16, 16, 3, 1, 1, seed=5)
    r1 = run_device("proposed", "conv", x, P, g, torch.bfloat16, 3, 1, 1)
    r2 = run_device("proposed", "conv", x, P, g, torch.bfloat16, 3, 1, 1)
    assert (r1[0] == r2[0]).all() and (r1[4] == r2[4]).all()
    for role in r1[3]:
        assert (r1[3][role] == r2[3][role]).all()


def test_c2_partitioned_step_fold_deterministic(monkeypatch):
    """C2 geometry: the wgrad3 / dgrad SM partition with wgrad3's in-kernel
    split-K fold (grid barrier + fixed-order slot sums) replays bit for bit, and
    agrees with the separate-kernel fold (QD_W3_NOFOLD=1; another summation
    order) to fp32 round-off; also under a CUDA graph replay."""
    from paper_2204_01701_b200 import neurons
    x, P, g = Q.synthetic_layer("proposed", "conv", 128, 64, 64, 32, 32, 3, 1, 1, seed=9)
    r1 = run_device("proposed", "conv", x, P, g, torch.bfloat16, 3, 1, 1)
    r2 = run_device("proposed", "conv", x, P, g, torch.bfloat16, 3, 1, 1)
    for role in r1[3]:
        assert (r1[3][role] == r2[3][role]).all(), role
    assert (r1[4] == r2[4]).all()
    monkeypatch.setenv("QD_W3_NOFOLD", "1")
    r3 = run_device("proposed", "conv", x, P, g, torch.bfloat16, 3, 1, 1)
    monkeypatch.delenv("QD_W3_NOFOLD")
    for role in r1[3]:
        assert Q.rel_err(r1[3][role], r3[3][role]) <= 1e-5, role
    # graph capture + two replays (the barrier slots reset themselves)
    dev = torch.device("cuda")
    spec = _spec("proposed", "conv", 64, 64, 3, 1, 1)
    xt = torch.as_tensor(x, device=dev).bfloat16().contiguous(memory_format=torch.channels_last)
    gt = torch.as_tensor(g, device=dev).bfloat16().contiguous(memory_format=torch.channels_last)
    params = {r: torch.as_tensor(v, dtype=torch.float32, device=dev) for r, v in P.items()}
    out = {}

    def step():
        y, cache = neurons.forward(spec, params, xt)
        grads, dx = neurons.symbolic_backward(spec, params, cache, gt)
        out["g"] = grads
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    reps = []
    for _ in range(2):
        graph.replay()
        torch.cuda.synchronize()
        reps.append({r: v.double().cpu().numpy().copy() for r, v in out["g"].items()})
    for role in reps[0]:
        assert (reps[0][role] == reps[1][role]).all(), role
        assert Q.rel_err(reps[0][role], r1[3][role]) <= 1e-5, role


def test_error_conventions_on_device():
    from paper_2204_01701_b200 import neurons
    from paper_2204_01701_b200.errors import DimensionError, IntegrityError
    dev = torch.device("cuda")
    s1 = _spec("t4", "fc", 3, 2)
    s2 = _spec("proposed", "fc", 3, 2)
    p1 = {"Wa": torch.randn(3, 2, device=dev), "Wb": torch.randn(3, 2, device=dev)}
    _, cache = neurons.forward(s1, p1, torch.randn(2, 3, device=dev))
    with pytest.raises(IntegrityError):
        neurons.symbolic_backward(s2, p1, cache, torch.zeros(2, 2, device=dev))
    with pytest.raises(IntegrityError):
        neurons.symbolic_backward(s1, p1, cache, torch.zeros(2, 5, device=dev))
    with pytest.raises(DimensionError):
        neurons.forward(s1, p1, torch.randn(2, 4, device=dev))
    sc = _spec("proposed", "conv", 1, 1, 5, 1, 0)
    pc = {r: torch.randn(*sh, device=dev) for r, sh in
          __import__("paper_2204_01701_b200.spec", fromlist=["x"]).param_shapes(sc).items()}
    with pytest.raises(DimensionError):
        neurons.forward(sc, pc, torch.randn(1, 1, 3, 3, device=dev))


def test_autograd_module_matches_functional():
    from paper_2204_01701_b200 import neurons
    from paper_2204_01701_b200.nn import QuadConv2d
    torch.manual_seed(0)
    m = QuadConv2d(64, 64, 3, 1, 1, device="cuda")
    x = torch.randn(2, 64, 8, 8, device="cuda", dtype=torch.bfloat16,
                    requires_grad=True).contiguous(memory_format=torch.channels_last)
    x.retain_grad()
    y = m(x)
    gy = torch.randn_like(y)
    y.backward(gy)
    y2, cache = neurons.forward(m.spec, m.params(), x.detach())
    grads, dx = neurons.symbolic_backward(m.spec, m.params(), cache, gy)
    assert torch.equal(y, y2)
    assert torch.equal(x.grad, dx)
    for role, g in grads.items():
        assert torch.equal(getattr(m, role).grad, g)


def test_kernels_launch_counter():
    from paper_2204_01701_b200 import _lib
    before = _lib.launch_count()
    x, P, g = Q.synthetic_layer("proposed", "conv", 2, 64, 64, 8, 8, 3, 1, 1)
    run_device("proposed", "conv", x, P, g, torch.bfloat16, 3, 1, 1)
    assert _lib.launch_count() > before


# depth-wise kind (qd_path == 2), every family that allows it: direct kernels and the
# shared-memory tiled ones
DW_CASES = [
    ("proposed", 4, 32, 14, 14, 3, 1, 1),
    ("proposed", 3, 24, 15, 13, 3, 2, 1),
    ("t4", 2, 16, 9, 9, 3, 1, 1),
    ("t2", 2, 16, 9, 9, 5, 1, 2),
    ("t3", 2, 16, 9, 9, 3, 1, 1),
    ("t2_linear", 2, 16, 9, 9, 3, 1, 1),
    ("t2and4", 2, 16, 10, 10, 3, 2, 1),
    ("first_order", 2, 16, 9, 9, 3, 1, 1),
    # shared-memory tiled kernels (r = 3, C % 32 == 0): tile edges, stride 2, pads 0 / 2
    ("proposed", 2, 64, 19, 37, 3, 1, 1),
    ("proposed", 2, 32, 17, 35, 3, 2, 1),
    ("t4", 2, 32, 9, 20, 3, 1, 1),
    ("t2", 2, 32, 11, 11, 3, 2, 1),
    ("t3", 2, 32, 9, 9, 3, 1, 1),
    ("t2_linear", 2, 32, 12, 18, 3, 1, 0),
    ("t2and4", 2, 32, 10, 10, 3, 2, 1),
    ("first_order", 2, 32, 9, 9, 3, 1, 2),
]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("case", DW_CASES, ids=[f"{c[0]}-c{c[2]}-{c[3]}x{c[4]}-k{c[5]}s{c[6]}p{c[7]}" for c in DW_CASES])
def test_dwconv_parity(case, dtype):
    fam, n, c, h, w, k, s, p = case
    x, P, g = Q.synthetic_layer(fam, "dwconv", n, c, c, h, w, k, s, p, seed=11, random_bias=True)
    path = check_against_oracle(fam, "dwconv", x, P, g, dtype, k, s, p)
    assert path == 2


# T1 families (fc, one output unit, full-rank quadratic weight): CUDA-core path
@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("fam", ["t1_pure", "t1_full", "t1and2"])
@pytest.mark.parametrize("n,c", [(64, 96), (300, 256)])
def test_t1_parity(fam, n, c, dtype):
    x, P, g = Q.synthetic_layer(fam, "fc", n, c, 1, seed=5)
    path = check_against_oracle(fam, "fc", x, P, g, dtype)
    assert path == 0


# fused SGD + pack
@pytest.mark.gpu
@pytest.mark.parametrize("family,kind,c,f,k", [("proposed", "conv", 64, 64, 3), ("t4", "conv", 64, 128, 3),
                                               ("t2_linear", "conv", 64, 64, 3), ("t2and4", "conv", 64, 64, 3),
                                               ("proposed", "fc", 96, 64, 1), ("first_order", "conv", 8, 16, 3),
                                               ("proposed", "conv", 40, 72, 5), ("t4", "fc", 100, 36, 1),
                                               ("proposed", "conv", 330, 340, 3)])
def test_quad_sgd_matches_torch_sgd_and_repack(family, kind, c, f, k):
    from paper_2204_01701_b200 import neurons
    from paper_2204_01701_b200.nn import QuadConv2d, QuadLinear
    from paper_2204_01701_b200.optim import QuadSGD
    torch.manual_seed(0)
    mk = (lambda: QuadConv2d(c, f, k, 1, k // 2, family=family, device="cuda")) if kind == "conv" else \
        (lambda: QuadLinear(c, f, family=family, device="cuda"))
    m1, m2 = mk(), mk()
    m2.load_state_dict(m1.state_dict())
    if kind == "conv":  # the nets move whole models to channels_last
        m1 = m1.to(memory_format=torch.channels_last)
    o1 = QuadSGD(m1, lr=0.05, momentum=0.9, weight_decay=5e-4)
    o2 = torch.optim.SGD(m2.parameters(), lr=0.05, momentum=0.9, weight_decay=5e-4, dampening=0.0)
    x = torch.randn((4, c, 10, 10) if kind == "conv" else (32, c), device="cuda")
    for it in range(3):
        for mod, opt in ((m1, o1), (m2, o2)):
            opt.zero_grad(set_to_none=True)
            y = mod(x.to(torch.bfloat16).contiguous(memory_format=torch.channels_last) if kind == "conv"
                    else x.to(torch.bfloat16))
            y.float().square().mean().backward()
            opt.step()
        for (n1, p1), (n2, p2) in zip(m1.named_parameters(), m2.named_parameters()):
            assert torch.allclose(p1, p2, rtol=1e-5, atol=1e-6), (it, n1)
    # the registered pack equals a fresh pack of the updated weights, bit for bit
    spec = m1.spec
    shape = (1, c) if kind == "fc" else (1, c, k, k)
    desc = neurons.make_desc(spec, shape, torch.bfloat16)
    roles = neurons.WEIGHT_ROLES[spec.family]
    reg = neurons._registered_pack(desc, [getattr(m1, r) for r in roles])
    assert reg is not None
    fresh = neurons._pack(spec, desc, {r: getattr(m1, r).detach().clone() for r in neurons.param_shapes(spec)})[0]
    torch.cuda.synchronize()
    assert torch.equal(reg, fresh)


# BN (+ReLU) fused around the quadratic conv
@pytest.mark.gpu
@pytest.mark.parametrize("family,kind,relu", [("proposed", "conv", True), ("proposed", "conv", False),
                                               ("t4", "conv", True), ("first_order", "conv", True),
                                               ("t2_linear", "conv", True), ("t2and4", "conv", True),
                                               ("proposed", "fc", True)])
def test_quadconvbn_fused_matches_reference_bn(family, kind, relu):
    from paper_2204_01701_b200.bn import QuadConvBN, _ref_batchnorm
    from paper_2204_01701_b200.nn import QuadConv2d, QuadFunction, QuadLinear
    from paper_2204_01701_b200.spec import param_shapes
    torch.manual_seed(3)
    c, f = 64, 64
    layer = QuadConv2d(c, f, 3, 1, 1, family=family, device="cuda") if kind == "conv" else \
        QuadLinear(c, f, family=family, device="cuda")
    mod = QuadConvBN(layer, relu=relu)
    with torch.no_grad():
        mod.weight.uniform_(0.5, 1.5)
        mod.bias.uniform_(-0.2, 0.2)
        for r in param_shapes(layer.spec):
            if r.startswith("b"):
                getattr(layer, r).uniform_(-0.1, 0.1)
    assert mod.fused()
    shape = (8, c, 12, 12) if kind == "conv" else (96, c)
    x0 = torch.randn(shape, device="cuda").to(torch.bfloat16)
    if kind == "conv":
        x0 = x0.contiguous(memory_format=torch.channels_last)
    gz = torch.randn((8, f, 12, 12) if kind == "conv" else (96, f), device="cuda").to(torch.bfloat16)
    rm0, rv0 = mod.bn.running_mean.clone(), mod.bn.running_var.clone()
    # fused
    x1 = x0.clone().requires_grad_(True)
    z1 = mod(x1)
    z1.backward(gz)
    g1 = {n: p.grad.clone() for n, p in mod.named_parameters()}
    rm1, rv1 = mod.bn.running_mean.clone(), mod.bn.running_var.clone()
    for p in mod.parameters():
        p.grad = None
    # reference composition: same layer kernels, reference BN with torch autograd
    x2 = x0.clone().requires_grad_(True)
    roles = tuple(param_shapes(layer.spec).keys())
    y = QuadFunction.apply(layer.spec, torch.bfloat16, x2, *[getattr(layer, r) for r in roles])
    rm2, rv2 = rm0.clone(), rv0.clone()
    z2 = _ref_batchnorm(y, mod.weight, mod.bias, rm2, rv2, 0.1, 1e-5, True)
    if relu:
        z2 = torch.relu(z2)
    z2.backward(gz)
    g2 = {n: p.grad.clone() for n, p in mod.named_parameters()}
    rel = lambda a, b: Q.rel_err(a.detach().double().cpu().numpy(), b.detach().double().cpu().numpy())  # noqa
    assert rel(z1, z2) <= 2e-2, rel(z1, z2)
    assert rel(x1.grad, x2.grad) <= 3e-2, rel(x1.grad, x2.grad)
    for n in g1:
        if n in ("layer.bc", "layer.b"):
            # a bias added right before BN has an exactly zero gradient (BN removes the
            # mean): the unfused path only sums bf16 rounding noise; the fused one (fp32 dy)
            # must cancel to round-off relative to the layer's other gradients
            other = max(float(g.abs().max()) for k, g in g1.items() if k.startswith("layer.W"))
            assert float(g1[n].abs().max()) <= 1e-3 * other, (n, float(g1[n].abs().max()), other)
            continue
        assert rel(g1[n], g2[n]) <= 3e-2, (n, rel(g1[n], g2[n]))
    assert torch.allclose(rm1, rm2, rtol=1e-3, atol=1e-4) and torch.allclose(rv1, rv2, rtol=1e-3, atol=1e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("family,relu", [("proposed", True), ("proposed", False), ("t4", True),
                                         ("first_order", True)])
def test_streaming_emit_matches_register_emit(family, relu, monkeypatch):
    """Large fused layers take the bulk-copy streaming D emission (bias gradients
    folded in-kernel): the same D as the register-streaming emit bit for bit
    (so dx and the weight gradients are identical), bias gradients to fp32
    summation-order round-off."""
    from paper_2204_01701_b200.bn import QuadConvBN
    from paper_2204_01701_b200.nn import QuadConv2d
    from paper_2204_01701_b200.spec import param_shapes
    torch.manual_seed(5)
    mod = QuadConvBN(QuadConv2d(64, 64, 3, 1, 1, family=family, device="cuda"), relu=relu)
    with torch.no_grad():
        mod.weight.uniform_(0.5, 1.5)
        mod.bias.uniform_(-0.2, 0.2)
        for r in param_shapes(mod.layer.spec):
            if r.startswith("b"):
                getattr(mod.layer, r).uniform_(-0.1, 0.1)
    x0 = torch.randn(64, 64, 64, 64, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    gz = torch.randn(64, 64, 64, 64, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    out = []
    for old in (False, True):
        if old:
            monkeypatch.setenv("QD_BN_OLD", "1")
        x1 = x0.clone().requires_grad_(True)
        for p in mod.parameters():
            p.grad = None
        mod(x1).backward(gz)
        out.append((x1.grad, {n: p.grad.clone() for n, p in mod.named_parameters()}))
    torch.cuda.synchronize()
    assert torch.equal(out[0][0], out[1][0])
    wmax = max(float(g.abs().max()) for n, g in out[0][1].items() if n.startswith("layer.W"))
    for n, g in out[0][1].items():
        if n in ("layer.bc", "layer.b"):  # exactly zero through BN: fold-order round-off only
            assert float(g.abs().max()) <= 1e-3 * wmax and float(out[1][1][n].abs().max()) <= 1e-3 * wmax, n
        elif n.startswith("layer.b"):  # bias: in-kernel fold vs bias_finish order
            assert torch.allclose(g, out[1][1][n], rtol=1e-4, atol=1e-5 * float(g.abs().max())), n
        else:
            assert torch.equal(g, out[1][1][n]), n


@pytest.mark.gpu
def test_quadconvbn_add_relu_matches_composition():
    """ResNet block tail relu(BN(layer(x)) + res) as one fused node (residual add
    and ReLU on the BN apply pass, mask z > 0 in the backward) vs the module's
    unfused composition on identical inputs and parameters."""
    import copy
    from paper_2204_01701_b200.bn import QuadConvBN
    from paper_2204_01701_b200.nn import QuadConv2d
    torch.manual_seed(6)
    mod = QuadConvBN(QuadConv2d(64, 64, 3, 1, 1, device="cuda"), relu=False)
    ref = copy.deepcopy(mod)
    x0 = torch.randn(4, 64, 12, 12, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    r0 = torch.randn(4, 64, 12, 12, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    gz = torch.randn(4, 64, 12, 12, device="cuda").bfloat16()
    x1, r1 = x0.clone().requires_grad_(True), r0.clone().requires_grad_(True)
    z1 = mod.forward_add_relu(x1, r1)
    z1.backward(gz)
    x2, r2 = x0.clone().requires_grad_(True), r0.clone().requires_grad_(True)
    import os
    os.environ["QD_NO_BNFUSE"] = "1"
    try:
        z2 = ref.forward_add_relu(x2, r2)
    finally:
        del os.environ["QD_NO_BNFUSE"]
    z2.backward(gz)
    rel = lambda a, b: Q.rel_err(a.detach().double().cpu().numpy(), b.detach().double().cpu().numpy())  # noqa
    assert rel(z1, z2) <= 2e-2, rel(z1, z2)
    # the ReLU masks agree except where bf16 rounding of BN(y) + res lands on the
    # other side of 0 (a max-norm error there is one whole gz value): the residual
    # gradient equals gz on the fused path's own mask exactly, and gradients are
    # compared in the Frobenius norm
    assert ((z1 > 0) != (z2 > 0)).float().mean().item() <= 5e-3
    assert torch.equal(r1.grad, gz * (z1.detach() > 0))
    fro = lambda a, b: ((a.double() - b.double()).norm() / b.double().norm()).item()  # noqa: E731
    assert fro(r1.grad, r2.grad) <= 5e-2, fro(r1.grad, r2.grad)
    assert fro(x1.grad, x2.grad) <= 5e-2, fro(x1.grad, x2.grad)
    g2 = dict(ref.named_parameters())
    for n, p in mod.named_parameters():
        if n == "layer.bc":  # exactly zero through BN: round-off only
            continue
        assert fro(p.grad, g2[n].grad) <= 5e-2, (n, fro(p.grad, g2[n].grad))
    assert torch.allclose(mod.bn.running_mean, ref.bn.running_mean, rtol=1e-3, atol=1e-4)


@pytest.mark.gpu
def test_quadconvbn_stride2_fused_path():
    """stride 2 on its own grid: BN(+ReLU) fused, D emitted on the stride-2
    output grid and consumed by the strided wgrad / parity-class dgrad"""
    from paper_2204_01701_b200.bn import QuadConvBN, _ref_batchnorm
    from paper_2204_01701_b200.nn import QuadConv2d, QuadFunction
    torch.manual_seed(4)
    layer = QuadConv2d(64, 128, 3, 2, 1, device="cuda")
    mod = QuadConvBN(layer, relu=True)
    x0 = torch.randn(4, 64, 16, 16, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    assert mod.fused(x0) and not mod.fused()
    gz = torch.randn(4, 128, 8, 8, device="cuda").bfloat16()
    x1 = x0.clone().requires_grad_(True)
    mod(x1).backward(gz)
    g1 = {n: p.grad.clone() for n, p in mod.named_parameters()}
    for p in mod.parameters():
        p.grad = None
    x2 = x0.clone().requires_grad_(True)
    y = QuadFunction.apply(layer.spec, torch.bfloat16, x2, *[getattr(layer, r) for r in ("Wa", "Wb", "Wc", "ba", "bb",
                                                                                           "bc")])
    z = torch.relu(_ref_batchnorm(y, mod.weight, mod.bias, torch.zeros(128, device="cuda"),
                                  torch.ones(128, device="cuda"), 0.1, 1e-5, True))
    z.backward(gz)
    rel = lambda a, b: Q.rel_err(a.detach().double().cpu().numpy(), b.detach().double().cpu().numpy())  # noqa
    assert rel(x1.grad, x2.grad) <= 3e-2
    for n, p in mod.named_parameters():
        if n in ("layer.bc",):
            continue
        assert rel(g1[n], p.grad) <= 3e-2, n


@pytest.mark.gpu
def test_memory_ledger_accounts_minimal_cache():
    """AUTO vs HYBRID retained bytes on QuadraVGG-16."""
    from paper_2204_01701_b200 import qnets
    from paper_2204_01701_b200.ledger import memory_ledger
    m = qnets.QuadraVGG16(10).cuda().to(memory_format=torch.channels_last)
    x = torch.randn(16, 3, 32, 32, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    led = memory_ledger(m, x)
    assert led.peak_auto > 0 and led.peak_hybrid > 0
    assert set(led.per_layer_auto) == set(led.per_layer_hybrid) and len(led.per_layer_hybrid) == 13
    # the symbolic node keeps exactly its minimal cache: a, b (neurons.cache_names; x is the
    # previous layer's output) + the BN input y + the output z, nothing else (no patches,
    # no intermediate sums); the op-by-op twin keeps at least as much
    from paper_2204_01701_b200.bn import QuadConvBN
    obytes = {}
    hooks = [mod.register_forward_hook(lambda md, i_, o, n=name: obytes.__setitem__(n, o.numel() * o.element_size()))
             for name, mod in m.named_modules() if isinstance(mod, QuadConvBN)]
    with torch.no_grad(), torch.autocast("cuda", dtype=torch.bfloat16):
        m(x)
    for h in hooks:
        h.remove()
    assert len(obytes) == 12
    for name, ob in obytes.items():
        got = led.per_layer_hybrid[name]
        # + batch statistics and allocator rounding (under one extra tensor in any run order)
        assert 4 * ob <= got < 5 * ob, (name, got, ob)
        assert led.per_layer_auto[name] >= 4 * ob, (name, led.per_layer_auto[name], ob)


# first-order pieces of the QuadraNet step on the library kernels
@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("geo", [(3, 2, 1, 2, 64, 23, 17), (2, 2, 0, 3, 16, 8, 8), (3, 1, 1, 1, 8, 5, 6),
                                 (2, 2, 0, 2, 512, 3, 5),
                                 (3, 2, 1, 2, 64, 24, 18), (3, 2, 1, 3, 16, 2, 4)])  # k3s2p1 even: 2x2-block bwd
def test_maxpool_matches_torch(geo, dtype):
    from paper_2204_01701_b200.pool import MaxPool2d
    k, s, p, n, c, h, w = geo
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(n, c, h, w, device="cuda", generator=g).to(dtype).contiguous(memory_format=torch.channels_last)
    x[0, :, 0, 0] = x[0, :, 0, 1]  # ties: the first maximum in scan order wins
    x1 = x.clone().requires_grad_(True)
    x2 = x.clone().requires_grad_(True)
    y1 = MaxPool2d(k, s, p)(x1)
    y2 = torch.nn.functional.max_pool2d(x2, k, s, p)
    assert torch.equal(y1, y2)
    gy = torch.randn(y1.shape, device="cuda", generator=g).to(dtype)
    y1.backward(gy)
    y2.backward(gy)
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-6
    assert Q.rel_err(x1.grad.double().cpu().numpy(), x2.grad.double().cpu().numpy()) <= tol


@pytest.mark.gpu
@pytest.mark.parametrize("relu", [False, True])
def test_bnact_matches_reference_bn(relu):
    from paper_2204_01701_b200.bn import BNAct2d, _ref_batchnorm
    g = torch.Generator(device="cuda").manual_seed(6)
    x = (torch.randn(4, 64, 9, 11, device="cuda", generator=g) * 2 + 0.5).to(torch.bfloat16)
    x = x.contiguous(memory_format=torch.channels_last)
    m = BNAct2d(64, relu=relu).cuda()
    with torch.no_grad():
        m.weight.uniform_(0.5, 1.5, generator=g)
        m.bias.uniform_(-0.5, 0.5, generator=g)
    ref_rm, ref_rv = m.running_mean.clone(), m.running_var.clone()
    x1 = x.clone().requires_grad_(True)
    z = m(x1)
    x2 = x.float().clone().requires_grad_(True)
    w2, b2 = m.weight.detach().clone().requires_grad_(True), m.bias.detach().clone().requires_grad_(True)
    z2 = _ref_batchnorm(x2, w2, b2, ref_rm, ref_rv, 0.1, 1e-5, True)
    z2 = torch.relu(z2) if relu else z2
    assert Q.rel_err(z.detach().double().cpu().numpy(), z2.detach().double().cpu().numpy()) <= 2e-2
    assert torch.allclose(m.running_mean, ref_rm, rtol=1e-4, atol=1e-5)
    assert torch.allclose(m.running_var, ref_rv, rtol=1e-4, atol=1e-5)  # biased variance (tensor.py:444)
    gz = torch.randn(z.shape, device="cuda", generator=g)
    z.backward(gz.to(z.dtype))
    z2.backward(gz)
    assert Q.rel_err(x1.grad.double().cpu().numpy(), x2.grad.double().cpu().numpy()) <= 2e-2
    assert Q.rel_err(m.weight.grad.double().cpu().numpy(), w2.grad.double().cpu().numpy()) <= 2e-2
    assert Q.rel_err(m.bias.grad.double().cpu().numpy(), b2.grad.double().cpu().numpy()) <= 2e-2
    assert int(m.num_batches_tracked) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("n,c,hw,dtype", [(2, 8, 3, torch.bfloat16), (4, 64, 9, torch.bfloat16),
                                          (128, 64, 56, torch.bfloat16), (32, 512, 7, torch.bfloat16),
                                          (3, 2048, 5, torch.bfloat16), (16, 256, 14, torch.float32),
                                          (5, 96, 7, torch.bfloat16), (2, 4096, 2, torch.bfloat16),
                                          (64, 64, 64, torch.float32)],
                         ids=["tiny", "small", "r18_64x56", "r18_512x7", "c2048", "fp32", "c96", "c4096", "fp32_big"])
def test_bn_kernels_vs_fp64_and_deterministic(n, c, hw, dtype):
    """BN (+ReLU) forward / backward across shapes and dtypes (the large ones take
    the streaming D emission, C = 96 / 4096 the scalar any-C kernels) against
    the fp64 composition: z, dx, dgamma, dbeta, running statistics; and
    bit-identical results on a second run (fixed-order folds)."""
    from paper_2204_01701_b200.bn import BNAct2d
    g = torch.Generator(device="cuda").manual_seed(n * c + hw)
    x = (torch.randn(n, c, hw, hw, device="cuda", generator=g) * 2 + 0.5).to(dtype)
    x = x.contiguous(memory_format=torch.channels_last)
    gz = torch.randn(x.shape, device="cuda", generator=g).to(dtype)
    m = BNAct2d(c, relu=True).cuda()
    with torch.no_grad():
        m.weight.uniform_(0.5, 1.5, generator=g)
        m.bias.uniform_(-0.5, 0.5, generator=g)
    rm0, rv0 = m.running_mean.clone(), m.running_var.clone()
    runs = []
    for _ in range(2):
        with torch.no_grad():
            m.running_mean.copy_(rm0)
            m.running_var.copy_(rv0)
        x1 = x.clone().requires_grad_(True)
        m.weight.grad = m.bias.grad = None
        z = m(x1)
        z.backward(gz)
        runs.append((z.detach(), x1.grad, m.weight.grad.clone(), m.bias.grad.clone(), m.running_mean.clone(),
                     m.running_var.clone()))
    for a, b in zip(*runs):
        assert torch.equal(a, b)
    z, dx, dw, db, rm, rv = runs[0]
    xd = x.double().requires_grad_(True)
    wd = m.weight.detach().double().requires_grad_(True)
    bd = m.bias.detach().double().requires_grad_(True)
    mean = xd.mean(dim=(0, 2, 3))
    var = xd.var(dim=(0, 2, 3), unbiased=False)
    t = wd.view(1, -1, 1, 1) * (xd - mean.view(1, -1, 1, 1)) * torch.rsqrt(var + 1e-5).view(1, -1, 1, 1) + \
        bd.view(1, -1, 1, 1)
    mask = (z > 0).double()  # the device's own ReLU mask (ties at 0 go either way)
    zr = t * mask
    zr.backward(gz.double())
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-4
    rel = lambda a, b: float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30))  # noqa
    assert rel(z, zr.detach()) <= (1e-2 if dtype == torch.bfloat16 else 1e-5)
    assert rel(dx, xd.grad) <= tol, rel(dx, xd.grad)
    assert rel(dw, wd.grad) <= tol, rel(dw, wd.grad)
    assert rel(db, bd.grad) <= tol, rel(db, bd.grad)
    assert torch.allclose(rm.double(), 0.9 * rm0.double() + 0.1 * mean.detach(), rtol=1e-4, atol=1e-5)
    assert torch.allclose(rv.double(), 0.9 * rv0.double() + 0.1 * var.detach(), rtol=1e-4, atol=1e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("family,k,s,p,c,w", [("first_order", 7, 2, 3, 3, 23), ("proposed", 3, 1, 1, 3, 23),
                                            ("t4", 3, 1, 1, 5, 23), ("proposed", 5, 2, 2, 2, 23),
                                            ("first_order", 7, 2, 3, 3, 240), ("proposed", 3, 1, 1, 3, 131)])
def test_im2col_conv_matches_torch_conv(family, k, s, p, c, w):
    """3-channel stems as one fc GEMM over im2col'd patches vs the conv computed
    by torch in fp32 from the same bf16 values (odd run starts at stride 1 with
    odd C; rows wider than one 112-pixel block)."""
    from paper_2204_01701_b200.im2col import Im2colConv2d
    import torch.nn.functional as F
    torch.manual_seed(2)
    m = Im2colConv2d(c, 64, k, s, p, family=family, bias=(family != "first_order")).cuda()
    with torch.no_grad():
        for name, t in m.named_parameters():
            if name.startswith("b"):
                t.uniform_(-0.2, 0.2)
    x = torch.randn(3, c, 19, w, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    y = m(x)
    assert y.is_contiguous(memory_format=torch.channels_last)
    gy = torch.randn(y.shape, device="cuda")
    y.backward(gy.to(y.dtype))
    xf = x.float()
    ref = {n: t.detach().bfloat16().float().requires_grad_(True) if t.dim() == 4 else t.detach().clone().requires_grad_(True)
           for n, t in m.named_parameters()}
    conv = lambda w: F.conv2d(xf, w, stride=s, padding=p)  # noqa: E731
    if family == "first_order":
        yr = conv(ref["W"])
    elif family == "t4":
        yr = conv(ref["Wa"]) * conv(ref["Wb"])
    else:
        a = conv(ref["Wa"]) + ref["ba"].view(1, -1, 1, 1)
        b = conv(ref["Wb"]) + ref["bb"].view(1, -1, 1, 1)
        yr = a * b + conv(ref["Wc"]) + ref["bc"].view(1, -1, 1, 1)
    yr.backward(gy)
    cv = lambda t: t.detach().double().cpu().numpy()  # noqa: E731
    assert Q.rel_err(cv(y), cv(yr)) <= 2e-2
    for n, t in m.named_parameters():
        assert Q.rel_err(cv(t.grad), cv(ref[n].grad)) <= 2e-2, n


def test_concurrent_host_threads_same_results():
    """Two host threads, each on its own CUDA stream, run the C2-shaped layer step
    (partitioned backward: side stream + fork/join events per thread and device)
    concurrently; each result equals the same step run alone, bit for bit."""
    import threading
    from paper_2204_01701_b200 import neurons
    dev = torch.device("cuda")
    spec = _spec("proposed", "conv", 64, 64, 3, 1, 1)
    cases = []
    for seed in (31, 32):
        x, P, g = Q.synthetic_layer("proposed", "conv", 32, 64, 64, 32, 32, 3, 1, 1, seed=seed)
        cases.append((torch.as_tensor(x, device=dev).bfloat16().contiguous(memory_format=torch.channels_last),
                      torch.as_tensor(g, device=dev).bfloat16().contiguous(memory_format=torch.channels_last),
                      {r: torch.as_tensor(v, dtype=torch.float32, device=dev) for r, v in P.items()}))

    def run(i, out, stream):
        xt, gt, params = cases[i]
        with torch.cuda.stream(stream):
            for _ in range(5):
                y, cache = neurons.forward(spec, params, xt)
                grads, dx = neurons.symbolic_backward(spec, params, cache, gt)
            stream.synchronize()
        out[i] = (y.clone(), dx.clone(), {k: v.clone() for k, v in grads.items()})

    alone = {}
    for i in range(2):
        run(i, alone, torch.cuda.Stream())
    conc = {}
    ths = [threading.Thread(target=run, args=(i, conc, torch.cuda.Stream())) for i in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for i in range(2):
        assert torch.equal(alone[i][0], conc[i][0]) and torch.equal(alone[i][1], conc[i][1])
        for k in alone[i][2]:
            assert torch.equal(alone[i][2][k], conc[i][2][k]), (i, k)


@pytest.mark.parametrize("shape,dtype", [((8, 64, 32, 32), torch.bfloat16), ((5, 128, 14, 14), torch.bfloat16),
                                         ((4, 64, 16, 16), torch.float32)])
def test_bn_statistics_from_fprop_epilogue(shape, dtype, monkeypatch):
    """BN forward statistics written by the layer's fprop epilogue (per 32-pixel
    warp mean / M2, Chan merge) vs the separate reduction pass over y: same batch
    mean / biased variance (running buffers) to fp32 round-off, same output z;
    the epilogue path launches no reduction kernel."""
    import copy
    from paper_2204_01701_b200.bn import QuadConvBN
    from paper_2204_01701_b200.nn import QuadConv2d
    from paper_2204_01701_b200 import neurons
    torch.manual_seed(8)
    n, c, h, w = shape
    m1 = QuadConvBN(QuadConv2d(c, c, 3, 1, 1, device="cuda", compute_dtype=dtype), relu=True)
    with torch.no_grad():
        for r in ("ba", "bb", "bc"):
            getattr(m1.layer, r).uniform_(-0.5, 1.5)  # non-zero channel means
    m2 = copy.deepcopy(m1)
    x = torch.randn(shape, device="cuda").to(dtype).contiguous(memory_format=torch.channels_last)
    assert neurons.bn_stats_rows(m1.layer.spec, shape, dtype) > 0
    monkeypatch.setenv("QD_BN_EPI", "1")
    z1, names1 = _kernel_names(lambda: m1(x))
    monkeypatch.setenv("QD_BN_EPI", "0")
    z2, names2 = _kernel_names(lambda: m2(x))
    assert "bn_stats_merge" in names1 and "bn_stats" not in names1, names1
    assert "bn_stats" in names2
    assert torch.allclose(m1.bn.running_mean, m2.bn.running_mean, rtol=1e-4, atol=1e-5)
    assert torch.allclose(m1.bn.running_var, m2.bn.running_var, rtol=1e-4, atol=1e-5)
    d = (z1.float() - z2.float()).abs()
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-4
    assert float(d.max()) <= tol * float(z2.float().abs().max()), float(d.max())


@pytest.mark.parametrize("case", [
    ("proposed", 128, 64, 64, 32, 32, 1, "QD_XFD"),    # C2: dgrad forms dy*b, dy*a itself
    ("proposed", 64, 128, 128, 28, 28, 1, "QD_XFD"),
    ("t2_linear", 8, 64, 64, 56, 56, 1, "QD_XFS"),     # fprop squares x in its transform warps
    ("t2_linear", 4, 128, 64, 20, 20, 2, "QD_XFS"),
    ("t2", 4, 64, 128, 16, 16, 1, "QD_XFS"),
    ("t2and4", 4, 64, 64, 24, 24, 1, "QD_XFS"),
], ids=lambda c: f"{c[0]}_{c[1]}x{c[2]}x{c[4]}s{c[6]}" if isinstance(c, tuple) else str(c))
def test_operand_transform_bit_identical(case, monkeypatch):
    """The conv2 operand-transform warps (x * x for the squared-input families,
    dy * b / dy * a for the dgrad's D blocks) write exactly the bf16 values the
    separate passes (square_vec / backward prologue) write, in the TMA's
    swizzled layout: every output and gradient is bit-identical to the default
    path. (Opt-in: measured slower.)"""
    fam, n, c, f, h, w, s, knob = case
    x, P, g = Q.synthetic_layer(fam, "conv", n, c, f, h, w, 3, s, 1, seed=11, random_bias=True)
    off = run_device(fam, "conv", x, P, g, torch.bfloat16, 3, s, 1)
    monkeypatch.setenv(knob, "1")
    on = run_device(fam, "conv", x, P, g, torch.bfloat16, 3, s, 1)
    monkeypatch.delenv(knob)
    assert on[5] == 1 and off[5] == 1
    assert (on[0] == off[0]).all(), "y"
    assert (on[4] == off[4]).all(), "dx"
    for role in on[3]:
        assert (on[3][role] == off[3][role]).all(), role


@pytest.mark.parametrize("shape", [(128, 512, 512, 7), (64, 256, 512, 14), (32, 128, 256, 8)])
def test_wgrad_pair_matches_single(shape, monkeypatch):
    """The CTA-pair v1 wgrad (M = 256 over two SMs, each holding half of the D
    boxes; the default where its cost model picks it) gives the single-CTA
    kernel's weight gradients (QD_WPAIR=0); both are checked against the oracle
    elsewhere."""
    n, c, f, hw = shape
    x, P, g = Q.synthetic_layer("proposed", "conv", n, c, f, hw, hw, 3, 1, 1, seed=3, random_bias=True)
    monkeypatch.setenv("QD_WPAIR", "0")
    base = run_device("proposed", "conv", x, P, g, torch.bfloat16, 3, 1, 1)
    monkeypatch.setenv("QD_WPAIR", "1")
    monkeypatch.setenv("QD_WPAIR_SMAX", "4")  # the split variants too
    pair = run_device("proposed", "conv", x, P, g, torch.bfloat16, 3, 1, 1)
    monkeypatch.delenv("QD_WPAIR")
    monkeypatch.delenv("QD_WPAIR_SMAX")
    for role in base[3]:
        assert Q.rel_err(pair[3][role], base[3][role]) <= 1e-5, role


def test_backward_on_a_fresh_host_thread():
    """The C ABI from a host thread whose first CUDA call it is (torch's autograd
    worker runs backward passes on such threads): the tensor-map encode binds the
    device's primary context instead of failing with CUDA_ERROR_INVALID_CONTEXT."""
    import threading
    from paper_2204_01701_b200 import neurons
    x, P, g = Q.synthetic_layer("proposed", "conv", 4, 64, 64, 16, 16, 3, 1, 1, seed=2)
    ref = run_device("proposed", "conv", x, P, g, torch.bfloat16, 3, 1, 1)
    spec = _spec("proposed", "conv", 64, 64, 3, 1, 1)
    dev = torch.device("cuda")
    params = {r: torch.as_tensor(v, dtype=torch.float32, device=dev) for r, v in P.items()}
    y, cache = neurons.forward(spec, params, torch.as_tensor(x, device=dev).bfloat16())
    gt = torch.as_tensor(g, device=dev).bfloat16()
    out, err = {}, []

    def work():
        try:
            grads, dx = neurons.symbolic_backward(spec, params, cache, gt)
            torch.cuda.synchronize()
            out.update(grads=grads, dx=dx)
        except Exception as e:  # noqa: BLE001 - reported below
            err.append(e)
    t = threading.Thread(target=work)
    t.start()
    t.join()
    assert not err, err
    assert (out["dx"].double().cpu().numpy() == ref[4]).all()
    for role in ref[3]:
        assert (out["grads"][role].double().cpu().numpy() == ref[3][role]).all(), role


@pytest.mark.parametrize("case", [("proposed", 64, 512, 512, 7, 1), ("t4", 32, 256, 512, 14, 2),
                                  ("first_order", 16, 128, 256, 28, 2), ("proposed", 4, 64, 64, 9, 1)],
                         ids=lambda c: f"{c[0]}_{c[1]}x{c[2]}x{c[4]}s{c[5]}")
def test_conv_gemm_pair_matches_single(case, monkeypatch):
    """The CTA-pair v1 conv GEMM (QD_CPAIR=1: M = 256 over two SMs, each holding
    half of the weight tile; fprop, stride-1 dgrad, stride-2 parity-class dgrad,
    split-K) reproduces the single-CTA kernel bit for bit (same MMAs per output
    row, same accumulation order)."""
    fam, n, c, f, hw, s = case
    x, P, g = Q.synthetic_layer(fam, "conv", n, c, f, hw, hw, 3, s, 1, seed=4, random_bias=True)
    base = run_device(fam, "conv", x, P, g, torch.bfloat16, 3, s, 1, flags=_lib_flag_v1())
    monkeypatch.setenv("QD_CPAIR", "1")
    pair = run_device(fam, "conv", x, P, g, torch.bfloat16, 3, s, 1, flags=_lib_flag_v1())
    monkeypatch.delenv("QD_CPAIR")
    assert (pair[0] == base[0]).all() and (pair[4] == base[4]).all()
    for role in base[3]:
        assert (pair[3][role] == base[3][role]).all(), role


def _lib_flag_v1():
    from paper_2204_01701_b200 import _lib
    return _lib.FLAG_TC_V1


@pytest.mark.parametrize("case", [("proposed", 6, 64, 64, 32, 32, 3), ("t4", 3, 64, 128, 17, 23, 3),
                                  ("proposed", 2, 64, 64, 20, 20, 5), ("proposed", 4, 128, 128, 14, 14, 3)],
                         ids=lambda c: f"{c[0]}_{c[1]}x{c[2]}x{c[4]}x{c[5]}k{c[6]}")
def test_grouped_b_stream_bit_identical(case, monkeypatch):
    """conv2 with streamed weights: one ring slot / barrier per channel block (all
    r*r taps, the default for 4 KB stages -- the fp32 split dgrad of 64-channel
    layers; QD_C2_BGROUP=1 everywhere it fits) issues the same MMAs in the same
    order as the per-tap ring (QD_C2_BGROUP=0), so every output is bit-identical;
    the grouped form is also checked against the fp64 oracle at 1e-4."""
    fam, n, c, f, h, w, k = case
    p = k // 2
    x, P, g = Q.synthetic_layer(fam, "conv", n, c, f, h, w, k, 1, p, seed=31, random_bias=True)
    monkeypatch.setenv("QD_C2_BGROUP", "0")
    base = run_device(fam, "conv", x, P, g, torch.float32, k, 1, p)
    monkeypatch.setenv("QD_C2_BGROUP", "1")
    grp = run_device(fam, "conv", x, P, g, torch.float32, k, 1, p)
    monkeypatch.delenv("QD_C2_BGROUP")
    dflt = run_device(fam, "conv", x, P, g, torch.float32, k, 1, p)
    assert base[5] == 3 and grp[5] == 3
    for other in (grp, dflt):
        assert (other[0] == base[0]).all() and (other[4] == base[4]).all()
        for role in base[3]:
            assert (other[3][role] == base[3][role]).all(), role
    monkeypatch.setenv("QD_C2_BGROUP", "1")
    assert check_against_oracle(fam, "conv", x, P, g, torch.float32, k, 1, p) == 3
