"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the reference is importable only here):

    python oracle/gen_golden.py            # writes tests/golden/*

It imports quadra from /root/reference/pkg/src (read-only, never copied),
evaluates ``neurons.forward`` / ``neurons.symbolic_backward`` and the
integer shape/count logic on seeded small cases, and stores inputs and
outputs under tests/golden/. The tests then pin both the oracle restatement
(oracle/quadra_oracle.py) and the product's host logic against these files;
nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _import_reference():
    sys.path.insert(0, REF_SRC)
    from quadra import neurons, tensor  # noqa: E402
    from quadra.autobuild import QuadraticLayerSpec  # noqa: E402
    from quadra import errors  # noqa: E402
    return neurons, tensor, QuadraticLayerSpec, errors


def spec_cases():
    fams = ["first_order", "t1_pure", "t1_full", "t1and2", "t2", "t3", "t4",
            "t2and4", "proposed", "bogus"]
    kinds = ["fc", "conv", "dwconv", "bad"]
    out = []
    for fam in fams:
        for kind in kinds:
            for (n, m) in [(3, 4), (4, 4), (1, 1), (0, 3), (64, 64), (5, 1)]:
                for (k, s, p) in [(1, 1, 0), (3, 1, 1), (3, 2, 1), (2, 1, 0),
                                  (0, 1, 0), (3, 0, 1), (3, 1, -1)]:
                    for act in ("none", "relu", "gelu"):
                        if act != "none" and (k, s, p) != (1, 1, 0):
                            continue
                        out.append(dict(kind=kind, family=fam, in_dim=n, out_dim=m,
                                        kernel=k, stride=s, pad=p, activation=act))
    return out


def gen_spec_golden(neurons, tensor, Spec, errors):
    rows = []
    for c in spec_cases():
        spec = Spec(**c)
        row = {"spec": c}
        try:
            neurons.validate_spec(spec)
            row["ok"] = True
        except Exception as e:  # noqa: BLE001
            row["ok"] = False
            row["error"] = type(e).__name__
            row["message"] = str(e)
            rows.append(row)
            continue
        row["describe"] = spec.describe()
        row["param_shapes"] = {k: list(v) for k, v in neurons.param_shapes(spec).items()}
        row["count_params"] = int(neurons.count_params(spec))
        row["count_weights"] = int(neurons.count_weights(spec))
        row["cache_names"] = list(neurons.cache_names(spec.family))
        if spec.kind == "fc":
            row["count_macs"] = int(neurons.count_macs(spec))
        else:
            macs = {}
            for hw in [(5, 5), (8, 7), (32, 32), (7, 7)]:
                shape = (spec.in_dim,) + hw
                try:
                    macs[f"{hw[0]}x{hw[1]}"] = int(neurons.count_macs(spec, shape))
                except Exception as e:  # noqa: BLE001
                    macs[f"{hw[0]}x{hw[1]}"] = type(e).__name__
            row["count_macs"] = macs
        rows.append(row)
    conv_sizes = []
    for size in range(1, 65):
        for r in range(1, 8):
            for stride in (1, 2, 3):
                for pad in (0, 1, 2, 3):
                    conv_sizes.append([size, r, stride, pad,
                                       int(tensor.conv_out_size(size, r, stride, pad))])
    return {"specs": rows, "conv_out_size": conv_sizes}


LAYER_CASES = [
    # (family, kind, n, c, f, h, w, k, s, p)
    ("proposed", "fc", 5, 7, 6, 1, 1, 1, 1, 0),
    ("t4", "fc", 5, 7, 6, 1, 1, 1, 1, 0),
    ("t2", "fc", 5, 7, 6, 1, 1, 1, 1, 0),
    ("first_order", "fc", 5, 7, 6, 1, 1, 1, 1, 0),
    ("proposed", "conv", 3, 3, 4, 5, 5, 3, 1, 1),   # test_forward_matches_formula_oracle geometry
    ("proposed", "conv", 3, 3, 4, 5, 5, 3, 2, 1),   # test_symbolic_matches_auto_tape geometry
    ("proposed", "conv", 2, 3, 2, 5, 5, 2, 1, 0),   # test_finite_difference_agreement geometry
    ("proposed", "conv", 2, 8, 16, 6, 7, 3, 1, 1),
    ("proposed", "conv", 2, 5, 3, 7, 6, 1, 1, 0),
    ("proposed", "conv", 2, 4, 4, 9, 9, 3, 2, 1),
    ("t4", "conv", 3, 3, 4, 5, 5, 3, 1, 1),
    ("t4", "conv", 3, 3, 4, 5, 5, 3, 2, 1),
    ("t4", "conv", 2, 3, 2, 5, 5, 2, 1, 0),
    ("t2", "conv", 3, 3, 4, 5, 5, 3, 1, 1),
    ("t2", "conv", 3, 3, 4, 5, 5, 3, 2, 1),
    ("t2", "conv", 2, 3, 2, 5, 5, 2, 1, 0),
    ("first_order", "conv", 3, 3, 4, 5, 5, 3, 1, 1),
    ("first_order", "conv", 3, 3, 4, 5, 5, 3, 2, 1),
]


def gen_layer_golden(neurons, tensor, Spec):
    T = tensor
    rng = np.random.default_rng(1234)
    files = []
    for idx, (fam, kind, n, c, f, h, w, k, s, p) in enumerate(LAYER_CASES):
        spec = Spec(kind=kind, family=fam, in_dim=c, out_dim=f, kernel=k, stride=s, pad=p)
        params = {role: rng.normal(size=shape)
                  for role, shape in neurons.param_shapes(spec).items()}
        x = rng.normal(size=(n, c) if kind == "fc" else (n, c, h, w))
        tp = {role: T.Tensor._wrap(v, is_param=True) for role, v in params.items()}
        y, cache = neurons.forward(spec, tp, T.Tensor._wrap(x))
        g = rng.normal(size=y.shape)
        grads, dx = neurons.symbolic_backward(spec, tp, cache, T.Tensor._wrap(g))
        rec = {"x": x, "g": g, "y": y.data, "dx": dx}
        for role, v in params.items():
            rec["P_" + role] = v
        for role, v in grads.items():
            rec["G_" + role] = v
        if cache.a is not None:
            rec["a"] = cache.a.data
            rec["b"] = cache.b.data
        name = f"layer_{idx:02d}_{fam}_{kind}_k{k}s{s}p{p}.npz"
        np.savez_compressed(os.path.join(OUT, name), **rec)
        files.append({"file": name, "family": fam, "kind": kind, "n": n, "c": c, "f": f,
                      "h": h, "w": w, "k": k, "s": s, "p": p})
    # t2_linear = reference t2 + bias-free reference first_order
    for idx, (kind, n, c, f, h, w, k, s, p) in enumerate([
            ("fc", 5, 7, 6, 1, 1, 1, 1, 0), ("conv", 3, 3, 4, 5, 5, 3, 1, 1),
            ("conv", 3, 3, 4, 5, 5, 3, 2, 1)]):
        s2 = Spec(kind=kind, family="t2", in_dim=c, out_dim=f, kernel=k, stride=s, pad=p)
        s1 = Spec(kind=kind, family="first_order", in_dim=c, out_dim=f, kernel=k,
                  stride=s, pad=p)
        wshape = neurons.param_shapes(s2)["Wa"]
        Wa = rng.normal(size=wshape)
        Wc = rng.normal(size=wshape)
        x = rng.normal(size=(n, c) if kind == "fc" else (n, c, h, w))
        xt = T.Tensor._wrap(x)
        y2, c2 = neurons.forward(s2, {"Wa": T.Tensor._wrap(Wa, is_param=True)}, xt)
        y1, c1 = neurons.forward(s1, {"W": T.Tensor._wrap(Wc, is_param=True),
                                      "b": T.Tensor._wrap(np.zeros(f), is_param=True)}, xt)
        g = rng.normal(size=y2.shape)
        g2, dx2 = neurons.symbolic_backward(s2, {"Wa": T.Tensor._wrap(Wa, is_param=True)},
                                            c2, T.Tensor._wrap(g))
        g1, dx1 = neurons.symbolic_backward(s1, {"W": T.Tensor._wrap(Wc, is_param=True),
                                                 "b": T.Tensor._wrap(np.zeros(f), is_param=True)},
                                            c1, T.Tensor._wrap(g))
        rec = {"x": x, "g": g, "y": y2.data + y1.data, "dx": dx2 + dx1,
               "P_Wa": Wa, "P_Wc": Wc, "G_Wa": g2["Wa"], "G_Wc": g1["W"]}
        name = f"layer_t2lin_{idx:02d}_{kind}_k{k}s{s}p{p}.npz"
        np.savez_compressed(os.path.join(OUT, name), **rec)
        files.append({"file": name, "family": "t2_linear", "kind": kind, "n": n, "c": c,
                      "f": f, "h": h, "w": w, "k": k, "s": s, "p": p})
    # round-1 additions: t3 and t2and4 (neurons.py:257-267, :355-379, :406-432) on their
    # own seed so the earlier files stay byte-identical
    rng2 = np.random.default_rng(4321)
    for idx, (fam, kind, n, c, f, h, w, k, s, p) in enumerate([
            ("t3", "fc", 5, 7, 6, 1, 1, 1, 1, 0),
            ("t3", "conv", 3, 3, 4, 5, 5, 3, 1, 1),
            ("t3", "conv", 3, 3, 4, 5, 5, 3, 2, 1),
            ("t3", "conv", 2, 3, 2, 5, 5, 2, 1, 0),
            ("t2and4", "fc", 5, 7, 6, 1, 1, 1, 1, 0),
            ("t2and4", "conv", 3, 3, 4, 5, 5, 3, 1, 1),
            ("t2and4", "conv", 3, 3, 4, 5, 5, 3, 2, 1),
            ("t2and4", "conv", 2, 3, 2, 5, 5, 2, 1, 0),
            # depth-wise kind (tensor.py:367-418) for every family that allows it
            ("proposed", "dwconv", 3, 4, 4, 6, 6, 3, 1, 1),
            ("proposed", "dwconv", 2, 3, 3, 7, 7, 3, 2, 1),
            ("t4", "dwconv", 2, 4, 4, 6, 5, 3, 1, 1),
            ("t2", "dwconv", 2, 4, 4, 6, 6, 3, 1, 1),
            ("t3", "dwconv", 2, 4, 4, 6, 6, 2, 1, 0),
            ("t2and4", "dwconv", 2, 4, 4, 6, 6, 3, 2, 1),
            ("first_order", "dwconv", 2, 4, 4, 6, 6, 3, 1, 1),
            # T1 families: fc, one output unit (neurons.py:58-65)
            ("t1_pure", "fc", 5, 7, 1, 1, 1, 1, 1, 0),
            ("t1_full", "fc", 5, 7, 1, 1, 1, 1, 1, 0),
            ("t1and2", "fc", 5, 7, 1, 1, 1, 1, 1, 0)]):
        spec = Spec(kind=kind, family=fam, in_dim=c, out_dim=f, kernel=k, stride=s, pad=p)
        params = {role: rng2.normal(size=shape)
                  for role, shape in neurons.param_shapes(spec).items()}
        x = rng2.normal(size=(n, c) if kind == "fc" else (n, c, h, w))
        tp = {role: T.Tensor._wrap(v, is_param=True) for role, v in params.items()}
        y, cache = neurons.forward(spec, tp, T.Tensor._wrap(x))
        g = rng2.normal(size=y.shape)
        grads, dx = neurons.symbolic_backward(spec, tp, cache, T.Tensor._wrap(g))
        rec = {"x": x, "g": g, "y": y.data, "dx": dx}
        for role, v in params.items():
            rec["P_" + role] = v
        for role, v in grads.items():
            rec["G_" + role] = v
        if cache.a is not None:
            rec["a"] = cache.a.data
            rec["b"] = cache.b.data
        name = f"layer_x{idx:02d}_{fam}_{kind}_k{k}s{s}p{p}.npz"
        np.savez_compressed(os.path.join(OUT, name), **rec)
        files.append({"file": name, "family": fam, "kind": kind, "n": n, "c": c, "f": f,
                      "h": h, "w": w, "k": k, "s": s, "p": p})
    return files


def gen_known_answers(neurons, tensor, Spec):
    """tests/test_neurons.py:117-132 scalar known answers, recomputed."""
    T = tensor
    spec = Spec(kind="fc", family="proposed", in_dim=1, out_dim=1)
    P = {"Wa": [[1.0]], "Wb": [[3.0]], "Wc": [[-1.0]], "ba": [0.0], "bb": [0.0], "bc": [0.0]}
    tp = {k: T.Tensor._wrap(np.asarray(v, dtype=np.float64), is_param=True) for k, v in P.items()}
    y, cache = neurons.forward(spec, tp, T.Tensor._wrap(np.asarray([[2.0]])))
    _, dx = neurons.symbolic_backward(spec, tp, cache, T.Tensor._wrap(np.asarray([[1.0]])))
    return {"scalar_params": P, "x": 2.0, "y": float(y.data[0, 0]), "dx": float(dx[0, 0])}


CKPT_CONFIG = """model tiny
layer conv family=proposed in=3 out=8 k=3 s=1 p=1 bn=1 act=relu
layer conv family=t4 in=8 out=8 k=3 s=2 p=1 bn=1 act=relu
layer dwconv family=proposed in=8 out=8 k=3 s=1 p=1 bn=0 act=relu
layer fc family=t2 in=2048 out=16 k=1 s=1 p=0 bn=1 act=relu
head fc in=16 classes=10
train epochs=1 batch=4 lr=0.1 seed=7 dataset=cifar10
"""


def gen_checkpoint():
    """A reference-written checkpoint (model.py:236-263) of a small chain model with
    batch norm, stride 2, dwconv and an fc after an implicit flatten, plus the
    reference's eval-mode logits on a fixed input -> tests/golden/ckpt_tiny*."""
    from quadra import autobuild, model as M  # noqa: E402
    from quadra import tensor as T  # noqa: E402
    cfg = autobuild.parse_config(CKPT_CONFIG)
    mdl = M.Model(cfg)
    rng = np.random.default_rng(99)
    for layer in mdl.layers:
        if layer.bn is not None:
            c = layer.bn.running_mean.shape[0]
            layer.bn.running_mean[:] = rng.normal(size=c) * 0.1
            layer.bn.running_var[:] = rng.uniform(0.5, 1.5, size=c)
            layer.bn.gamma = T.Tensor._wrap(rng.uniform(0.5, 1.5, size=c), is_param=True)
            layer.bn.beta = T.Tensor._wrap(rng.normal(size=c) * 0.1, is_param=True)
    path = os.path.join(OUT, "ckpt_tiny")
    M.save_checkpoint(mdl, path)
    x = rng.normal(size=(4, 3, 32, 32))
    logits = mdl.forward(T.Tensor._wrap(x), tape=None, train=False).data
    np.savez_compressed(os.path.join(OUT, "ckpt_tiny_io.npz"), x=x, logits=logits,
                        serialized=np.array(autobuild.serialize_config(cfg)))


def main():
    os.makedirs(OUT, exist_ok=True)
    neurons, tensor, Spec, errors = _import_reference()
    spec_g = gen_spec_golden(neurons, tensor, Spec, errors)
    with open(os.path.join(OUT, "spec_golden.json"), "w") as fh:
        json.dump(spec_g, fh, separators=(",", ":"))
    files = gen_layer_golden(neurons, tensor, Spec)
    known = gen_known_answers(neurons, tensor, Spec)
    gen_checkpoint()
    with open(os.path.join(OUT, "index.json"), "w") as fh:
        json.dump({"generated_from": REF_SRC, "layers": files, "known_answers": known},
                  fh, indent=1)
    print(f"wrote {len(spec_g['specs'])} spec rows, {len(files)} layer cases -> {OUT}")


if __name__ == "__main__":
    main()
