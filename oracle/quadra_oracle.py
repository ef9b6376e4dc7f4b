"""CPU oracle for the quadratic-layer hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and
only as the checker or as the timed CPU baseline. The product path
(``paper_2204_01701_b200``) never imports it and has no CPU fallback.

It restates, in float64 numpy, the reference algorithm of
/root/reference/pkg/src/quadra (a pure-Python numpy library):
patch-matrix (im2col) lowering, BLAS GEMMs, the scatter-add adjoint
(col2im), the per-family forward and the closed-form backward, term by term
in the reference's accumulation order. Each function cites the reference
lines it follows.

Parity pin: tests/test_oracle_golden.py checks every function here against
golden vectors produced by running the reference itself
(oracle/gen_golden.py -> tests/golden/*.npz, committed), so this restatement
is pinned to the reference's own outputs; the golden cases include the
reference tests' known answers (scalar y=10, dx=11; Wa=0 => linear; dy=0 =>
zero gradients).

The ``t2_linear`` family (``Wa (x*x) + Wc x``) is not a reference family;
its oracle is the sum of the reference's ``t2`` and bias-free
``first_order``, both of which are pinned.
"""

from __future__ import annotations

import numpy as np


def conv_out_size(size, r, stride, pad):
    """tensor.py:279-280."""
    return (size + 2 * pad - r) // stride + 1


def im2col(x, r, stride, pad):
    """Patch matrix (N*oh*ow, C*r*r), K order (c, dy, dx); tensor.py:283-295."""
    n, c, h, w = x.shape
    oh = conv_out_size(h, r, stride, pad)
    ow = conv_out_size(w, r, stride, pad)
    img = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    col = np.empty((n, c, r, r, oh, ow))
    for dy in range(r):
        ymax = dy + stride * oh
        for dx in range(r):
            xmax = dx + stride * ow
            col[:, :, dy, dx, :, :] = img[:, :, dy:ymax:stride, dx:xmax:stride]
    return col.transpose(0, 4, 5, 1, 2, 3).reshape(n * oh * ow, c * r * r), oh, ow


def col2im(dcol, x_shape, r, stride, pad, oh, ow):
    """Scatter-add adjoint of im2col; tensor.py:298-310."""
    n, c, h, w = x_shape
    dcol = dcol.reshape(n, oh, ow, c, r, r).transpose(0, 3, 4, 5, 1, 2)
    img = np.zeros((n, c, h + 2 * pad, w + 2 * pad))
    for dy in range(r):
        ymax = dy + stride * oh
        for dx in range(r):
            xmax = dx + stride * ow
            img[:, :, dy:ymax:stride, dx:xmax:stride] += dcol[:, :, dy, dx, :, :]
    if pad:
        return img[:, :, pad:pad + h, pad:pad + w]
    return img


def conv_forward(x, w, stride, pad):
    """tensor.py:313-320."""
    f = w.shape[0]
    col, oh, ow = im2col(x, w.shape[2], stride, pad)
    out = col @ w.reshape(f, -1).T
    return np.ascontiguousarray(out.reshape(x.shape[0], oh, ow, f).transpose(0, 3, 1, 2))


def conv_backward(g, col, w, x_shape, stride, pad):
    """tensor.py:323-331: (dW, dX)."""
    n, f, oh, ow = g.shape
    r = w.shape[2]
    dmat = np.ascontiguousarray(g.transpose(0, 2, 3, 1)).reshape(-1, f)
    dw = (dmat.T @ col).reshape(w.shape)
    dcol = dmat @ w.reshape(f, -1)
    return dw, col2im(dcol, x_shape, r, stride, pad, oh, ow)


def dw_im2col(x, r, stride, pad):
    """Per-channel patch matrix (N, C, r*r, oh*ow); tensor.py:367-380."""
    n, c, h, w = x.shape
    oh = conv_out_size(h, r, stride, pad)
    ow = conv_out_size(w, r, stride, pad)
    img = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    col = np.empty((n, c, r * r, oh * ow))
    for dy in range(r):
        ymax = dy + stride * oh
        for dx in range(r):
            xmax = dx + stride * ow
            col[:, :, dy * r + dx, :] = img[:, :, dy:ymax:stride, dx:xmax:stride].reshape(n, c, -1)
    return col, oh, ow


def dwconv_forward(x, w, stride, pad):
    """tensor.py:383-388: per-channel cross-correlation, w (C, r, r)."""
    n, c = x.shape[:2]
    col, oh, ow = dw_im2col(x, w.shape[-1], stride, pad)
    y = np.einsum("nckl,ck->ncl", col, w.reshape(c, -1)).reshape(n, c, oh, ow)
    return np.ascontiguousarray(y)


def dwconv_backward(g, col, w, x_shape, stride, pad):
    """tensor.py:391-405: (dW, dX)."""
    n, c, oh, ow = g.shape
    r = w.shape[-1]
    gmat = g.reshape(n, c, -1)
    dw = np.einsum("ncl,nckl->ck", gmat, col).reshape(w.shape)
    dcol = np.einsum("ncl,ck->nckl", gmat, w.reshape(c, -1))
    img = np.zeros((n, c, x_shape[2] + 2 * pad, x_shape[3] + 2 * pad))
    for dy in range(r):
        ymax = dy + stride * oh
        for dx in range(r):
            xmax = dx + stride * ow
            img[:, :, dy:ymax:stride, dx:xmax:stride] += dcol[:, :, dy * r + dx, :].reshape(n, c, oh, ow)
    if pad:
        return dw, img[:, :, pad:pad + x_shape[2], pad:pad + x_shape[3]]
    return dw, img


class Geometry:
    """kind + (kernel, stride, pad); mirrors the spec fields the math needs."""

    def __init__(self, kind, kernel=1, stride=1, pad=0):
        self.kind, self.kernel, self.stride, self.pad = kind, kernel, stride, pad


def _lin(geo, x, w):
    """neurons.py:223-228 (fc: x @ W with W (in, out); conv: im2col GEMM)."""
    if geo.kind == "fc":
        return x @ w
    if geo.kind == "dwconv":
        return dwconv_forward(x, w, geo.stride, geo.pad)
    return conv_forward(x, w, geo.stride, geo.pad)


def _bias(geo, y, b):
    """neurons.py:231-232."""
    return y + b if geo.kind == "fc" else y + b[None, :, None, None]


def forward(family, geo, P, x):
    """neurons.py:235-276. Returns (y, a, b); a/b are None unless cached."""
    x = np.asarray(x, dtype=np.float64)
    a = b = None
    if family == "first_order":
        y = _bias(geo, _lin(geo, x, P["W"]), P["b"])
    elif family == "t1_pure":                             # :245-247
        v = x @ P["Wq"]
        y = (v * x).sum(axis=1, keepdims=True)
    elif family == "t1_full":                             # :248-250
        v = x @ P["Wq"]
        y = (v * x).sum(axis=1, keepdims=True) + x @ P["Wb"]
    elif family == "t1and2":                              # :251-254
        s = x * x
        v = x @ P["Wq"]
        y = (v * x).sum(axis=1, keepdims=True) + s @ P["Wb"]
    elif family == "t2":
        y = _lin(geo, x * x, P["Wa"])
    elif family == "t3":                                  # :257-259
        av = _lin(geo, x, P["Wa"])
        y = av * av
    elif family == "t4":
        a = _lin(geo, x, P["Wa"])
        b = _lin(geo, x, P["Wb"])
        y = a * b
    elif family == "t2and4":                              # :264-267
        a = _lin(geo, x, P["Wa"])
        b = _lin(geo, x, P["Wb"])
        y = a * b + _lin(geo, x * x, P["Wc"])
    elif family == "t2_linear":
        # reference t2 (neurons.py:255-256) + bias-free first_order (:242-244)
        y = _lin(geo, x * x, P["Wa"]) + _lin(geo, x, P["Wc"])
    elif family == "proposed":
        a = _bias(geo, _lin(geo, x, P["Wa"]), P["ba"])
        b = _bias(geo, _lin(geo, x, P["Wb"]), P["bb"])
        y = a * b + _bias(geo, _lin(geo, x, P["Wc"]), P["bc"])
    else:
        raise ValueError(f"oracle does not cover family {family!r}")
    return y, a, b


def _grads(geo, g, col, w, x_shape):
    """neurons.py:283-286 (conv / dwconv)."""
    if geo.kind == "dwconv":
        return dwconv_backward(g, col, w, x_shape, geo.stride, geo.pad)
    return conv_backward(g, col, w, x_shape, geo.stride, geo.pad)


def _col(geo, x):
    """neurons.py:289-292 (_make_col)."""
    if geo.kind == "dwconv":
        return dw_im2col(x, geo.kernel, geo.stride, geo.pad)[0]
    return im2col(x, geo.kernel, geo.stride, geo.pad)[0]


def symbolic_backward(family, geo, P, x, a, b, g):
    """neurons.py:295-445, same terms in the same order. Returns (grads, dx)."""
    xa = np.asarray(x, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    grads = {}
    if geo.kind == "fc":
        if family == "first_order":                      # :316-319
            grads["b"] = g.sum(axis=0)
            grads["W"] = xa.T @ g
            dx = g @ P["W"].T
        elif family == "t2":                             # :349-354
            s = xa * xa
            grads["Wa"] = s.T @ g
            ds = g @ P["Wa"].T
            t = ds * xa
            dx = t + t
        elif family == "t1_pure":                        # :320-326
            v = xa @ P["Wq"]
            dh = np.broadcast_to(g, xa.shape).copy()
            dv = dh * xa
            dx = dh * v
            grads["Wq"] = xa.T @ dv
            dx = dx + dv @ P["Wq"].T
        elif family == "t1_full":                        # :327-335
            v = xa @ P["Wq"]
            grads["Wb"] = xa.T @ g
            dx = g @ P["Wb"].T
            dh = np.broadcast_to(g, xa.shape).copy()
            dv = dh * xa
            dx = dx + dh * v
            grads["Wq"] = xa.T @ dv
            dx = dx + dv @ P["Wq"].T
        elif family == "t1and2":                         # :336-348
            s = xa * xa
            v = xa @ P["Wq"]
            grads["Wb"] = s.T @ g
            ds = g @ P["Wb"].T
            dh = np.broadcast_to(g, xa.shape).copy()
            dv = dh * xa
            dx = dh * v
            grads["Wq"] = xa.T @ dv
            dx = dx + dv @ P["Wq"].T
            t = ds * xa
            dx = dx + t
            dx = dx + t
        elif family == "t3":                             # :355-360
            av = xa @ P["Wa"]
            t = g * av
            da = t + t
            grads["Wa"] = xa.T @ da
            dx = da @ P["Wa"].T
        elif family == "t2and4":                         # :368-379
            s = xa * xa
            grads["Wc"] = s.T @ g
            ds = g @ P["Wc"].T
            t = ds * xa
            dx = t + t
            da = g * b
            db = g * a
            grads["Wb"] = xa.T @ db
            dx = dx + db @ P["Wb"].T
            grads["Wa"] = xa.T @ da
            dx = dx + da @ P["Wa"].T
        elif family == "t4":                             # :361-367
            da = g * b
            db = g * a
            grads["Wb"] = xa.T @ db
            dx = db @ P["Wb"].T
            grads["Wa"] = xa.T @ da
            dx = dx + da @ P["Wa"].T
        elif family == "t2_linear":                      # t2 :349-354 + first_order :316-319
            s = xa * xa
            grads["Wa"] = s.T @ g
            ds = g @ P["Wa"].T
            t = ds * xa
            dx = t + t
            grads["Wc"] = xa.T @ g
            dx = dx + g @ P["Wc"].T
        elif family == "proposed":                       # :380-391
            grads["bc"] = g.sum(axis=0)
            grads["Wc"] = xa.T @ g
            dx = g @ P["Wc"].T
            da = g * b
            db = g * a
            grads["bb"] = db.sum(axis=0)
            grads["Wb"] = xa.T @ db
            dx = dx + db @ P["Wb"].T
            grads["ba"] = da.sum(axis=0)
            grads["Wa"] = xa.T @ da
            dx = dx + da @ P["Wa"].T
        else:
            raise ValueError(family)
        return grads, dx

    x_shape = xa.shape
    r, s_, p_ = geo.kernel, geo.stride, geo.pad
    if family == "first_order":                          # :396-399
        grads["b"] = g.sum(axis=(0, 2, 3))
        col = _col(geo, xa)
        grads["W"], dx = _grads(geo, g, col, P["W"], x_shape)
    elif family == "t2":                                 # :400-405
        s = xa * xa
        col_s = _col(geo, s)
        grads["Wa"], ds = _grads(geo, g, col_s, P["Wa"], x_shape)
        t = ds * xa
        dx = t + t
    elif family == "t3":                                 # :406-411
        col = _col(geo, xa)
        av = _lin(geo, xa, P["Wa"])
        t = g * av
        da = t + t
        grads["Wa"], dx = _grads(geo, da, col, P["Wa"], x_shape)
    elif family == "t2and4":                             # :420-432
        s = xa * xa
        col_s = _col(geo, s)
        grads["Wc"], ds = _grads(geo, g, col_s, P["Wc"], x_shape)
        t = ds * xa
        dx = t + t
        col = _col(geo, xa)
        da = g * b
        db = g * a
        grads["Wb"], dxb = _grads(geo, db, col, P["Wb"], x_shape)
        dx = dx + dxb
        grads["Wa"], dxa = _grads(geo, da, col, P["Wa"], x_shape)
        dx = dx + dxa
    elif family == "t4":                                 # :412-419
        col = _col(geo, xa)
        da = g * b
        db = g * a
        grads["Wb"], dxb = _grads(geo, db, col, P["Wb"], x_shape)
        dx = dxb
        grads["Wa"], dxa = _grads(geo, da, col, P["Wa"], x_shape)
        dx = dx + dxa
    elif family == "t2_linear":
        s = xa * xa
        col_s = _col(geo, s)
        grads["Wa"], ds = _grads(geo, g, col_s, P["Wa"], x_shape)
        t = ds * xa
        dx = t + t
        col = _col(geo, xa)
        grads["Wc"], dxl = _grads(geo, g, col, P["Wc"], x_shape)
        dx = dx + dxl
    elif family == "proposed":                           # :433-444
        grads["bc"] = g.sum(axis=(0, 2, 3))
        col = _col(geo, xa)
        grads["Wc"], dx = _grads(geo, g, col, P["Wc"], x_shape)
        da = g * b
        db = g * a
        grads["bb"] = db.sum(axis=(0, 2, 3))
        grads["Wb"], dxb = _grads(geo, db, col, P["Wb"], x_shape)
        dx = dx + dxb
        grads["ba"] = da.sum(axis=(0, 2, 3))
        grads["Wa"], dxa = _grads(geo, da, col, P["Wa"], x_shape)
        dx = dx + dxa
    else:
        raise ValueError(family)
    return grads, dx


def rel_err(a, b):
    """max|a-b| / max(max|a|, max|b|) -- reference tests/oracles.py:98-102."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    denom = max(np.abs(a).max(initial=0.0), np.abs(b).max(initial=0.0), 1e-30)
    return float(np.abs(a - b).max(initial=0.0) / denom)


def conv2d_loops(x, w, stride, pad):
    """Six-loop direct convolution (reference tests/oracles.py:28-46) for the
    exhaustive geometry sweep; small shapes only."""
    n, c, h, wd = x.shape
    f, _, r, _ = w.shape
    oh = (h + 2 * pad - r) // stride + 1
    ow = (wd + 2 * pad - r) // stride + 1
    xp = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    out = np.zeros((n, f, oh, ow))
    for yi in range(oh):
        for xi in range(ow):
            patch = xp[:, :, yi * stride:yi * stride + r, xi * stride:xi * stride + r]
            out[:, :, yi, xi] = np.einsum("ncij,fcij->nf", patch, w)
    return out


# ---------------------------------------------------------------------------
# seeded synthetic inputs; shared by tests and bench
# ---------------------------------------------------------------------------

def synthetic_layer(family, kind, n, c, f, h=1, w=1, r=1, stride=1, pad=0,
                    seed=0, kaiming_uniform=True, random_bias=False):
    """x ~ N(0,1) (seed), weights Kaiming-uniform (seed+1), dy ~ N(0,1) (seed+2).

    fp64 arrays in the reference layouts: x NCHW (or (N, C) for fc), conv
    weights (F, C, r, r), fc weights (C, F), biases (F,).
    """
    rx = np.random.default_rng(seed)
    rw = np.random.default_rng(seed + 1)
    rg = np.random.default_rng(seed + 2)
    if kind == "fc":
        x = rx.standard_normal((n, c))
        wshape = (c, f)
        fan = c
        oh = ow = None
    elif kind == "dwconv":
        x = rx.standard_normal((n, c, h, w))
        wshape = (c, r, r)
        fan = r * r
        oh = conv_out_size(h, r, stride, pad)
        ow = conv_out_size(w, r, stride, pad)
    else:
        x = rx.standard_normal((n, c, h, w))
        wshape = (f, c, r, r)
        fan = c * r * r
        oh = conv_out_size(h, r, stride, pad)
        ow = conv_out_size(w, r, stride, pad)
    roles = {"first_order": ("W",), "t2": ("Wa",), "t3": ("Wa",), "t4": ("Wa", "Wb"),
             "t2_linear": ("Wa", "Wc"), "t2and4": ("Wa", "Wb", "Wc"),
             "proposed": ("Wa", "Wb", "Wc"), "t1_pure": ("Wq",), "t1_full": ("Wq", "Wb"),
             "t1and2": ("Wq", "Wb")}[family]
    if family.startswith("t1"):  # one output unit, full-rank quadratic weight (neurons.py:90-95)
        x = rx.standard_normal((n, c))
        P = {}
        bound = np.sqrt(6.0 / c)
        P["Wq"] = rw.uniform(-bound, bound, size=(c, c)) / np.sqrt(c)
        if family != "t1_pure":
            P["Wb"] = rw.uniform(-bound, bound, size=(c, 1))
        g = rg.standard_normal((n, 1))
        return x, P, g
    P = {}
    bound = np.sqrt(6.0 / fan)
    for role in roles:
        if kaiming_uniform:
            P[role] = rw.uniform(-bound, bound, size=wshape)
        else:
            P[role] = rw.standard_normal(wshape)
    bias_roles = {"first_order": ("b",), "proposed": ("ba", "bb", "bc")}.get(family, ())
    for role in bias_roles:
        P[role] = rw.standard_normal(f) if random_bias else np.zeros(f)
    g = rg.standard_normal((n, f) if kind == "fc" else (n, f, oh, ow))
    return x, P, g
