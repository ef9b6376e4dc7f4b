"""Cached-bytes ledger: AUTO vs HYBRID back-propagation.

Three views of the same question (paper: 26.7 % saving):

* ``reference_ledger(cfg, batch)`` -- the REFERENCE's own accounting, restated:
  a tape that keeps every non-parameter array a node references (AUTO run,
  each quadratic layer composed op by op with its three im2col patch matrices,
  model.py:170-230, tensor.py:355-364) against need-based retention with each
  quadratic layer as one symbolic node keeping x, a, b (HYBRID run,
  tensor.py:100-115, neurons.py:466-477); peaks = the forward's cumulative
  bytes (Tape.record, tensor.py:151-174). Pinned to the reference's tape by
  tests/test_ledger.py.
* ``device_ledger(model, x)`` -- torch.cuda.memory_allocated around real
  forwards on the device: the HYBRID node (x, a, b), the same node in
  recompute mode (x only), and the reference's AUTO composition run through
  torch autograd with explicit im2col patches (F.unfold + matmul per branch).
* ``memory_ledger(model, x)`` -- the op-by-op twin through cuDNN (no patch
  matrices), kept for the QuadraNets.

The reference accounts the arrays its tape retains for the backward pass per
layer, once with every op recorded separately (AUTO) and once with each
quadratic layer as one symbolic node that keeps only its minimal cache
(HYBRID), trainer.py:68-110 / :287-340 (paper: 26.7% saving).

Here both modes are real executions measured with torch.cuda.memory_allocated:
HYBRID is the model as built (each quadratic layer is one autograd node keeping
x, a, b -- neurons.cache_names); AUTO swaps every quadratic layer for the same
algebra written op by op in torch (convolutions through cuDNN, products and sums
as separate autograd ops), so autograd keeps whatever each op needs. Note the
reference's AUTO cost is dominated by its cached im2col patch matrices, which a
cuDNN composition does not keep -- the torch numbers show what the symbolic
node saves on THIS stack, not a re-run of the numpy accounting.
"""

from __future__ import annotations

import copy
from dataclasses import dataclass

import torch
import torch.nn.functional as Fnn
from torch import nn

from .bn import QuadConvBN
from .nn import _QuadBase


class AutoQuad(nn.Module):
    """A quadratic layer recorded op by op (reference model.py:170-230 _compose_auto).
    Weights are held as bf16 copies made once (parameters are not part of the
    ledger, like the reference's tape accounting, tensor.py:175-183)."""

    def __init__(self, q: _QuadBase):
        super().__init__()
        self.spec = q.spec
        for name, p in q.named_parameters():  # bf16 leaves that require grad: autograd records every op
            self.register_parameter(name, nn.Parameter(p.detach().to(torch.bfloat16).contiguous()))

    def _lin(self, x, w):
        s = self.spec
        if s.kind == "fc":
            return x @ w
        if s.kind == "dwconv":
            return Fnn.conv2d(x, w.unsqueeze(1), stride=s.stride, padding=s.pad, groups=s.in_dim)
        return Fnn.conv2d(x, w, stride=s.stride, padding=s.pad)

    def _addb(self, y, b):
        return y + (b if self.spec.kind == "fc" else b.view(1, -1, 1, 1))

    def forward(self, x):
        fam, lin = self.spec.family, self._lin
        x = x.to(torch.bfloat16)
        if fam == "first_order":
            return self._addb(lin(x, self.W), self.b)
        if fam == "t2":
            return lin(x * x, self.Wa)
        if fam == "t3":
            a = lin(x, self.Wa)
            return a * a
        if fam == "t4":
            return lin(x, self.Wa) * lin(x, self.Wb)
        if fam == "t2_linear":
            return lin(x * x, self.Wa) + lin(x, self.Wc)
        if fam == "t2and4":
            return lin(x, self.Wa) * lin(x, self.Wb) + lin(x * x, self.Wc)
        if fam == "proposed":
            a = self._addb(lin(x, self.Wa), self.ba)
            b = self._addb(lin(x, self.Wb), self.bb)
            return a * b + self._addb(lin(x, self.Wc), self.bc)
        raise ValueError(f"AUTO composition does not cover {fam}")


class _AutoQuadBN(nn.Module):
    def __init__(self, m: QuadConvBN):
        super().__init__()
        self.q = AutoQuad(m.layer)
        self.bn = nn.BatchNorm2d(m.layer.spec.out_dim) if m.layer.spec.kind != "fc" else \
            nn.BatchNorm1d(m.layer.spec.out_dim)
        self.bn.to(m.weight.device)
        self.relu = m.relu

    def forward(self, x):
        z = self.bn(self.q(x))
        return torch.relu(z) if self.relu else z


def to_auto(model: nn.Module) -> nn.Module:
    """Deep copy with every quadratic layer recorded op by op (parameters shared)."""
    def swap(mod):
        for name, child in list(mod.named_children()):
            if isinstance(child, QuadConvBN):
                setattr(mod, name, _AutoQuadBN(child))
            elif isinstance(child, _QuadBase):
                setattr(mod, name, AutoQuad(child))
            else:
                swap(child)
    auto = copy.copy(model)
    auto.__dict__ = dict(model.__dict__)
    auto._modules = {k: copy.deepcopy(v) if not isinstance(v, (_QuadBase, QuadConvBN)) else v
                     for k, v in model._modules.items()}
    swap(auto)
    return auto


@dataclass
class MemoryLedger:
    per_layer_auto: dict
    per_layer_hybrid: dict
    peak_auto: int
    peak_hybrid: int

    @property
    def saving_fraction(self):
        return 0.0 if self.peak_auto == 0 else 1.0 - self.peak_hybrid / self.peak_auto


def _retained(model, x, layers):
    """Bytes held after the forward (graph alive), total and per listed layer."""
    per = {}
    hooks = []
    state = {}
    for tag, mod in layers:
        hooks.append(mod.register_forward_pre_hook(lambda m, i, t=tag: state.__setitem__(t, torch.cuda.memory_allocated())))
        hooks.append(mod.register_forward_hook(lambda m, i, o, t=tag: per.__setitem__(
            t, torch.cuda.memory_allocated() - state[t])))
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    with torch.autocast("cuda", dtype=torch.bfloat16):
        out = model(x)
    torch.cuda.synchronize()
    total = torch.cuda.memory_allocated() - base
    for h in hooks:
        h.remove()
    del out
    return total, per


def _register_packs(model):
    """Packed weights made once and registered on the weights (what optim.QuadSGD
    does every step), so neither mode counts parameter-derived buffers."""
    from . import neurons
    for m in model.modules():
        if isinstance(m, _QuadBase) and m.spec.kind != "dwconv" and not m.spec.family.startswith("t1"):
            shape = (1, m.spec.in_dim) if m.spec.kind == "fc" else (1, m.spec.in_dim, m.spec.kernel, m.spec.kernel)
            desc = neurons.make_desc(m.spec, shape, m.compute_dtype)
            roles = neurons.WEIGHT_ROLES[m.spec.family]
            wpack = neurons._pack(m.spec, desc, m.params())[0]
            neurons.register_pack(desc, [getattr(m, r) for r in roles], wpack)


def memory_ledger(model: nn.Module, x: torch.Tensor) -> MemoryLedger:
    """Forward-retained activation bytes of `model` (HYBRID) and of its op-by-op twin
    (AUTO); parameters and parameter-derived buffers excluded in both."""
    _register_packs(model)
    def quad_layers(m):
        return [(n, c) for n, c in m.named_modules() if isinstance(c, (_QuadBase, QuadConvBN, AutoQuad, _AutoQuadBN))
                and not isinstance(getattr(c, "_parent_quad", None), object)]
    model.train()
    from .im2col import Im2colConv2d  # 3-channel stems: the same module in both modes
    hyb_layers = [(n, c) for n, c in model.named_modules() if isinstance(c, (QuadConvBN, Im2colConv2d)) or
                  (isinstance(c, _QuadBase) and not n.endswith(".layer"))]
    th, ph = _retained(model, x, hyb_layers)
    auto = to_auto(model)
    auto_layers = [(n, c) for n, c in auto.named_modules() if isinstance(c, (_AutoQuadBN, Im2colConv2d)) or
                   (isinstance(c, AutoQuad) and not n.endswith(".q"))]
    ta, pa = _retained(auto, x, auto_layers)
    return MemoryLedger(per_layer_auto=pa, per_layer_hybrid=ph, peak_auto=ta, peak_hybrid=th)


# ---------------------------------------------------------------------------
# the reference's accounting (tensor.py:137-185), restated for chain configs
# ---------------------------------------------------------------------------
class _Tape:
    """Byte accounting of the reference Tape for one mode: each node adds the
    bytes of the arrays its rule keeps that no earlier node kept (by identity)."""

    NEEDS = {"matmul": ("a", "b"), "bias_add": (), "bias_add_ch": (), "add": (), "hadamard": ("a", "b"),
             "relu": ("out",), "conv2d": ("patch",), "batchnorm": ("xhat", "inv_std"), "reshape": (),
             "softmax_ce": ("probs",)}

    def __init__(self, mode, itemsize):
        self.mode, self.itemsize = mode, itemsize
        self.seen = set()
        self.per_layer = {}
        self._ids = 0

    def new(self, nelem):
        self._ids += 1
        return (self._ids, int(nelem))

    def record(self, op, arrays, tag, retain=None):
        names = tuple(arrays) if self.mode == "auto" else (retain if retain is not None else self.NEEDS[op])
        added = 0
        for nm in names:
            t = arrays[nm]
            if t is None or t[0] in self.seen:  # None = a parameter (never counted)
                continue
            self.seen.add(t[0])
            added += t[1] * self.itemsize
        self.per_layer[tag] = self.per_layer.get(tag, 0) + added


def _quad_layer(tp, spec, x, batch, hw, tag):
    """Record one quadratic layer; returns its output array (id, elems)."""
    from .spec import conv_out_size
    fam = spec.family
    if spec.kind == "fc":
        out_n = batch * spec.out_dim
        patch_n = None
    else:
        oh = conv_out_size(hw[0], spec.kernel, spec.stride, spec.pad)
        ow = conv_out_size(hw[1], spec.kernel, spec.stride, spec.pad)
        out_n = batch * spec.out_dim * oh * ow
        patch_n = batch * oh * ow * spec.in_dim * spec.kernel * spec.kernel
    if tp.mode == "hybrid" and fam != "first_order":
        y = tp.new(out_n)
        arrays = {"out": y, "x": x}
        if fam in ("proposed", "t4", "t2and4"):
            arrays["a"], arrays["b"] = tp.new(out_n), tp.new(out_n)
        tp.record("quad", arrays, tag, retain=cache_names(fam))
        return y

    def lin(inp):
        o = tp.new(out_n)
        if spec.kind == "fc":
            tp.record("matmul", {"out": o, "a": inp, "b": None}, tag)
        else:
            tp.record("conv2d", {"out": o, "x": inp, "w": None, "patch": tp.new(patch_n)}, tag)
        return o

    def addb(inp):
        o = tp.new(out_n)
        tp.record("bias_add" if spec.kind == "fc" else "bias_add_ch", {"out": o, "x": inp, "b": None}, tag)
        return o

    def op2(op, a, b):
        o = tp.new(out_n)
        tp.record(op, {"out": o, "a": a, "b": b}, tag)
        return o
    if fam == "first_order":
        return addb(lin(x))
    if fam == "t4":
        return op2("hadamard", lin(x), lin(x))
    if fam == "proposed":
        a = addb(lin(x))
        b = addb(lin(x))
        h = op2("hadamard", a, b)
        return op2("add", h, addb(lin(x)))
    raise ValueError(f"reference_ledger: family {fam} not modelled")


def cache_names(family):
    from .spec import cache_names as cn
    return cn(family)


def reference_ledger(cfg, batch, input_shape=None, itemsize=8):
    """(AUTO run, HYBRID run) of the reference's accounting for a chain config:
    each a dict with per-layer bytes and the peak (the forward's total; the
    backward only releases). ``itemsize`` 8 = the reference's float64."""
    from .model import DATASET_SHAPES, _head_spec
    from .spec import output_spatial
    c, h, w = input_shape or DATASET_SHAPES[cfg.train.dataset]
    out = {}
    for mode in ("auto", "hybrid"):
        tp = _Tape(mode, itemsize)
        x = tp.new(batch * c * h * w)
        feat, hw = c, (h, w)
        for i, spec in enumerate(list(cfg.layers) + [_head_spec(cfg.head)]):
            tag = f"L{i}" if i < len(cfg.layers) else "head"
            if spec.kind == "fc" and hw is not None:  # implicit flatten (model.py:129-132)
                flat = tp.new(batch * feat * hw[0] * hw[1])
                tp.record("reshape", {"out": flat, "x": x}, tag)
                x, hw = flat, None
            y = _quad_layer(tp, spec, x, batch, hw, tag)
            ny = y[1]
            if spec.kind != "fc":
                hw = output_spatial(spec, hw)
            if getattr(spec, "batchnorm", False):
                z = tp.new(ny)
                tp.record("batchnorm", {"out": z, "x": y, "gamma": None, "beta": None, "xhat": tp.new(ny),
                                        "inv_std": tp.new(spec.out_dim)}, tag)
                y = z
            if getattr(spec, "activation", "none") == "relu":
                r = tp.new(ny)
                tp.record("relu", {"out": r, "x": y}, tag)
                y = r
            x, feat = y, spec.out_dim
        loss = tp.new(1)
        tp.record("softmax_ce", {"out": loss, "logits": x, "probs": tp.new(batch * cfg.head.classes)}, "loss")
        out[mode] = {"per_layer": tp.per_layer, "peak": sum(tp.per_layer.values())}
    return out["auto"], out["hybrid"]


# ---------------------------------------------------------------------------
# device measurement on chain models (torch.cuda.memory_allocated)
# ---------------------------------------------------------------------------
class AutoQuadPatches(nn.Module):
    """The reference's AUTO composition of a quadratic layer (model.py:170-230)
    through torch autograd, each convolution as im2col (F.unfold) + matmul like
    the reference's conv2d (tensor.py:313-320), so every branch materialises its
    own patch matrix; bf16 weight copies (parameters are not in the ledger)."""

    def __init__(self, q: _QuadBase):
        super().__init__()
        self.spec = q.spec
        for name, p in q.named_parameters():
            self.register_parameter(name, nn.Parameter(p.detach().to(torch.bfloat16).contiguous()))

    def _lin(self, x, w):
        s = self.spec
        if s.kind == "fc":
            return x @ w
        n, _, h, wd = x.shape
        oh = (h + 2 * s.pad - s.kernel) // s.stride + 1
        ow = (wd + 2 * s.pad - s.kernel) // s.stride + 1
        patch = Fnn.unfold(x, s.kernel, padding=s.pad, stride=s.stride)  # (N, C r r, OH OW)
        y = w.reshape(w.shape[0], -1) @ patch
        return y.reshape(n, w.shape[0], oh, ow)

    def _addb(self, y, b):
        return y + (b if self.spec.kind == "fc" else b.view(1, -1, 1, 1))

    def forward(self, x):
        fam, lin = self.spec.family, self._lin
        x = x.to(torch.bfloat16)
        if fam == "first_order":
            return self._addb(lin(x, self.W), self.b)
        if fam == "t4":
            return lin(x, self.Wa) * lin(x, self.Wb)
        if fam == "proposed":
            a = self._addb(lin(x, self.Wa), self.ba)
            b = self._addb(lin(x, self.Wb), self.bb)
            return a * b + self._addb(lin(x, self.Wc), self.bc)
        raise ValueError(f"AUTO composition does not cover {fam}")


def _forward_bytes(model, x):
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    with torch.autocast("cuda", dtype=torch.bfloat16):
        out = model(x)
    torch.cuda.synchronize()
    held = torch.cuda.memory_allocated() - base
    del out
    return held


def device_ledger(model, x):
    """Bytes the forward leaves allocated for the backward on the device, for a
    chain model (model.QuadraModel): {"hybrid": x, a, b per node, "recompute":
    x per node, "auto_patches": the reference's AUTO composition with patch
    matrices}. Parameters and packed weights are excluded (registered first)."""
    import copy as _copy
    _register_packs(model)
    model.train()
    res = {"hybrid": _forward_bytes(model, x)}
    quads = [m for m in model.modules() if isinstance(m, _QuadBase)]
    for q in quads:
        q.recompute_ab = True
    try:
        res["recompute"] = _forward_bytes(model, x)
    finally:
        for q in quads:
            q.recompute_ab = False
    auto = _copy.deepcopy(model)
    def swap(mod):
        for name, child in list(mod.named_children()):
            if isinstance(child, QuadConvBN):
                bn = nn.BatchNorm2d(child.layer.spec.out_dim) if child.layer.spec.kind != "fc" else \
                    nn.BatchNorm1d(child.layer.spec.out_dim)
                seq = nn.Sequential(AutoQuadPatches(child.layer), bn.to(child.weight.device))
                if child.relu:
                    seq.append(nn.ReLU())
                setattr(mod, name, seq)
            elif isinstance(child, _QuadBase):
                setattr(mod, name, AutoQuadPatches(child))
            else:
                swap(child)
    swap(auto)
    res["auto_patches"] = _forward_bytes(auto, x)
    return res
