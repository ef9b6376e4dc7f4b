"""Parity of the EXACT timed paths at the benchmarked configurations.

Every case runs the kernel sequence ``bench.py`` times (public API, the same
shapes and dtypes; for C2 the whole step captured in a CUDA graph and
replayed, with the wgrad3 / dgrad SM partition and wgrad3's in-kernel split-K
fold, asserted through the library's launch log) and compares ALL outputs --
y, the a / b cache, dx, every dW and db -- with the fp64 oracle on identical
(dtype-rounded) inputs, at full batch. The oracle runs in batch chunks; the
chunk sums of dW / db equal the full-batch sums up to fp64 round-off.

Tolerances: rel_err (reference tests/oracles.py:98-102) <= 2e-2 for bf16,
<= 1e-4 for fp32 (BASELINE.json north_star).
"""
import numpy as np
import pytest
import torch

from oracle import quadra_oracle as Q

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


def _spec(family, kind, c, f, k=1, s=1, p=0):
    from paper_2204_01701_b200.spec import QuadraticLayerSpec
    return QuadraticLayerSpec(kind=kind, family=family, in_dim=c, out_dim=f, kernel=k, stride=s, pad=p)


def _q(a, dtype):
    return torch.as_tensor(a).to(dtype).to(torch.float64).numpy()


def _cv(t):
    return None if t is None else t.detach().to(torch.float64).cpu().numpy()


def _kernel_log(fn):
    from paper_2204_01701_b200 import _lib
    lib = _lib.load()
    torch.cuda.synchronize()
    lib.qd_profile(1)
    try:
        fn()
        torch.cuda.synchronize()
        names = [n for n, _ in _lib.profile_read()]
    finally:
        lib.qd_profile(0)
    return names


def device_step(family, kind, x, P, g, dtype, k, s, p, graph=False):
    """forward + symbolic_backward through the public API (bench.py run_ours
    compute()), optionally captured as a CUDA graph and replayed twice."""
    from paper_2204_01701_b200 import neurons
    n, c = x.shape[:2]
    f = g.shape[1]
    spec = _spec(family, kind, c, f, k, s, p)
    dev = torch.device("cuda")
    xt = torch.as_tensor(x, device=dev).to(dtype)
    gt = torch.as_tensor(g, device=dev).to(dtype)
    if kind != "fc":
        xt = xt.contiguous(memory_format=torch.channels_last)
        gt = gt.contiguous(memory_format=torch.channels_last)
    params = {r: torch.as_tensor(v, dtype=torch.float32, device=dev) for r, v in P.items()}
    out = {}

    def step():
        y, cache = neurons.forward(spec, params, xt, dtype=dtype)
        grads, dx = neurons.symbolic_backward(spec, params, cache, gt)
        out.update(y=y, a=cache.a, b=cache.b, grads=grads, dx=dx)

    names = _kernel_log(step)
    if graph:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream().wait_stream(side)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            step()
        # poison the static outputs, then replay: every value must come from the replay
        for t in [out["y"], out["dx"]] + list(out["grads"].values()):
            t.fill_(float("nan"))
        gr.replay()
        gr.replay()
    torch.cuda.synchronize()
    res = {"y": _cv(out["y"]), "a": _cv(out["a"]), "b": _cv(out["b"]), "dx": _cv(out["dx"]),
           "grads": {r: _cv(v) for r, v in out["grads"].items()}}
    return res, names


def oracle_chunked(family, geo, Pq, xq, gq, a_dev, b_dev, chunk):
    """fp64 oracle over batch chunks; the backward uses the kernel's own (rounded)
    a, b cache like the reference backward uses its cache."""
    n = xq.shape[0]
    ys, as_, bs, dxs, gsum = [], [], [], [], None
    for i in range(0, n, chunk):
        sl = slice(i, min(n, i + chunk))
        ry, ra, rb = Q.forward(family, geo, Pq, xq[sl])
        ys.append(ry)
        if ra is not None:
            as_.append(ra)
            bs.append(rb)
        rg, rdx = Q.symbolic_backward(family, geo, Pq, xq[sl],
                                      None if a_dev is None else a_dev[sl],
                                      None if b_dev is None else b_dev[sl], gq[sl])
        dxs.append(rdx)
        gsum = rg if gsum is None else {r: gsum[r] + v for r, v in rg.items()}
    cat = lambda L: np.concatenate(L) if L else None  # noqa: E731
    return cat(ys), cat(as_), cat(bs), cat(dxs), gsum


def check_full(family, kind, n, c, f, h, w, k, s, p, dtype, seed=0, random_bias=False, graph=False,
               chunk=16):
    x, P, g = Q.synthetic_layer(family, kind, n, c, f, h, w, k, s, p, seed=seed, random_bias=random_bias)
    xq, gq = _q(x, dtype), _q(g, dtype)
    Pq = {r: (_q(v, dtype) if not r.startswith("b") else _q(v, torch.float32)) for r, v in P.items()}
    dev, names = device_step(family, kind, xq, P, gq, dtype, k, s, p, graph=graph)
    ry, ra, rb, rdx, rg = oracle_chunked(family, Q.Geometry(kind, k, s, p), Pq, xq, gq, dev["a"], dev["b"],
                                         chunk)
    tol = TOL[dtype]
    errs = {"y": Q.rel_err(dev["y"], ry), "dx": Q.rel_err(dev["dx"], rdx)}
    if ra is not None:
        errs["a"] = Q.rel_err(dev["a"], ra)
        errs["b"] = Q.rel_err(dev["b"], rb)
    assert set(dev["grads"]) == set(rg)
    for r in rg:
        errs[r] = Q.rel_err(dev["grads"][r], rg[r])
    bad = {k_: v for k_, v in errs.items() if not v <= tol}
    assert not bad, (bad, errs)
    return names, errs


# ---- C2: the bench's default workload, exactly as timed ----------------------
@pytest.mark.parametrize("random_bias", [False, True], ids=["bench_inputs", "random_bias"])
def test_c2_bf16_timed_step_graph_vs_oracle(random_bias):
    """BASELINE config 2 (128x64x32x32 -> 64, 3x3/s1/p1, bf16): the captured,
    replayed step of bench.py; the partitioned wgrad3 folds its split-K
    partials in-kernel (no separate fold launches)."""
    names, errs = check_full("proposed", "conv", 128, 64, 64, 32, 32, 3, 1, 1, torch.bfloat16, seed=0,
                             random_bias=random_bias, graph=True)
    assert names.count("conv2") == 2 and "wgrad3" in names and "prologue" in names, names
    assert "wsum" not in names and "bwd_finish" not in names, names


def test_c2_fp32_full_batch_vs_oracle():
    """BASELINE config 2 in fp32 at N = 128 (the fp32 bench workload c2_fp32), 1e-4."""
    check_full("proposed", "conv", 128, 64, 64, 32, 32, 3, 1, 1, torch.float32, seed=0, graph=True)


def test_c1_fp32_graph_vs_oracle():
    """BASELINE config 1 (fc 256x512 -> 512, fp32) through the captured step, 1e-4."""
    check_full("proposed", "fc", 256, 512, 512, 1, 1, 1, 1, 0, torch.float32, seed=0, graph=True, chunk=256)


# ---- C5: the neuron-variant sweep at its configuration (N = 64) --------------
C5 = [(fam, c, hw) for fam in ("proposed", "t4", "t2_linear") for c, hw in ((64, 56), (128, 28), (256, 14),
                                                                            (512, 7))]


@pytest.mark.parametrize("fam,c,hw", C5, ids=[f"{a}-{b}x{d}" for a, b, d in C5])
def test_c5_variant_full_config_vs_oracle(fam, c, hw):
    check_full(fam, "conv", 64, c, c, hw, hw, 3, 1, 1, torch.bfloat16, seed=0, chunk=8)


# ---- QuadraResNet-18 stride-2 layers at the net's batch (128) ----------------
S2 = [(64, 128, 56), (128, 256, 28), (256, 512, 14)]


@pytest.mark.parametrize("c,f,hw", S2, ids=[f"{a}to{b}@{d}" for a, b, d in S2])
def test_resnet_stride2_layers_batch128_vs_oracle(c, f, hw):
    names, _ = check_full("proposed", "conv", 128, c, f, hw, hw, 3, 2, 1, torch.bfloat16, seed=0,
                          random_bias=True, chunk=8)
    assert "conv_gemm" in names or "conv2" in names, names


# ---- C5 cross product off the diagonal (SURVEY.md §8(d) "full 4 x 4") ---------
# The kernel plan (halo tiles, resident weights, wgrad form, split-K) follows the
# layer shape (C, H, W), so every off-diagonal point of the measured grid
# (profiles/r2f_c5_grid.txt) is checked here at a small batch the fp64 oracle
# finishes in seconds; the diagonal runs at the full N = 64 above.
C5_OFF = [(c, hw) for c in (64, 128, 256, 512) for hw in (56, 28, 14, 7)
          if (c, hw) not in ((64, 56), (128, 28), (256, 14), (512, 7))]
C5_OFF_CASES = [(fam, c, hw) for fam in ("proposed", "t4", "t2_linear") for c, hw in C5_OFF]


@pytest.mark.parametrize("fam,c,hw", C5_OFF_CASES, ids=[f"{a}-{b}x{d}" for a, b, d in C5_OFF_CASES])
def test_c5_grid_off_diagonal_vs_oracle(fam, c, hw):
    n = 4 if hw >= 28 else 8
    check_full(fam, "conv", n, c, c, hw, hw, 3, 1, 1, torch.bfloat16, seed=0, random_bias=True, chunk=1)
