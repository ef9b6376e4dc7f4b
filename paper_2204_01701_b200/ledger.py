"""Cached-bytes ledger: AUTO vs HYBRID back-propagation.

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
