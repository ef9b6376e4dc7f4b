"""torch.nn modules over the quadratic-layer kernels.

The reference records a quadratic layer as ONE symbolic tape node whose
backward is the closed form (neurons.py:466-477, tensor.py:601-609); here that
node is a ``torch.autograd.Function`` whose backward calls
``neurons.symbolic_backward`` -- the paper's own "hybrid back-propagation"
design. Parameters keep the reference role names
(``Wa, Wb, Wc, ba, bb, bc``) and layouts (conv (F, C, r, r); fc (in, out)),
mirroring the paper's ``qua.type#()`` module API.
"""

from __future__ import annotations

import math

import torch
from torch import nn

from . import neurons
from .dp import grad_ready, take_grad
from .spec import QuadraticLayerSpec, fan_in, param_shapes, validate_device_spec


def grad_sinks(named, needs):
    """{name: bucket view} for the parameters whose gradients the library may write
    straight into their data-parallel buckets (dp.take_grad); ``named`` maps
    name -> parameter, ``needs`` name -> whether autograd wants its gradient"""
    out = {}
    for k, p in named.items():
        if needs.get(k):
            t = take_grad(p)
            if t is not None:
                out[k] = t
    return out


def settle_sinks(named, sinks, grads):
    """After the kernels that wrote them are enqueued: mark the sunk parameters
    ready and return the gradients autograd still has to accumulate (None for a
    sunk one). A sink the library did not use (its buffer was replaced) goes back
    through autograd, which adds into the zeroed bucket and fires the hook."""
    res = {}
    for k, g in grads.items():
        t = sinks.get(k)
        if t is not None and g is t:
            grad_ready(named[k])
            res[k] = None
        else:
            res[k] = g
    return res


class QuadFunction(torch.autograd.Function):
    """y = layer(x; params) with the closed-form backward (one tape node)."""

    @staticmethod
    def forward(ctx, spec, dtype, x, *tensors):
        roles = tuple(param_shapes(spec).keys())
        params = dict(zip(roles, tensors))
        dtype, recompute = neurons.split_opts(dtype)
        y, cache = neurons.forward(spec, params, x, dtype=dtype, recompute=recompute)
        ctx.spec, ctx.roles, ctx.params, ctx.cache = spec, roles, params, cache
        ctx.x_dtype = x.dtype
        return y

    @staticmethod
    def backward(ctx, gy):
        want_dx = ctx.needs_input_grad[2]
        # bias gradients only when some bias is trained (a constant zero bias, e.g.
        # a bias-free first-order stem, skips the bias reduction pass)
        bro = neurons.BIAS_ROLES.get(ctx.spec.family, ())
        want_db = any(ctx.needs_input_grad[3 + i] for i, r in enumerate(ctx.roles) if r in bro)
        sinks = grad_sinks(ctx.params, {r: ctx.needs_input_grad[3 + i] for i, r in enumerate(ctx.roles)})
        grads, dx = neurons.symbolic_backward(ctx.spec, ctx.params, ctx.cache, gy,
                                              want_dx=want_dx, want_db=want_db, out=sinks)
        grads = settle_sinks(ctx.params, sinks, grads)
        if dx is not None and dx.dtype != ctx.x_dtype:
            dx = dx.to(ctx.x_dtype)
        ctx.cache = None
        return (None, None, dx) + tuple(grads.get(r) for r in ctx.roles)


def quadratic(spec, params, x, dtype=None):
    """Autograd-tracked layer call; ``params`` maps role -> tensor."""
    roles = tuple(param_shapes(spec).keys())
    return QuadFunction.apply(spec, dtype, x, *[params[r] for r in roles])


def _reset(module, spec, generator=None, init="reference"):
    """'reference': neurons.py:132-147 semantics (normal sqrt(2/fan_in), Wb x0.1,
    zero bias); 'kaiming_uniform': U(+-sqrt(6/fan_in)) for every weight, zero
    bias (BASELINE.json configs)."""
    fi = fan_in(spec)
    with torch.no_grad():
        for role in param_shapes(spec):
            p = getattr(module, role)
            if role.startswith("b"):
                p.zero_()
            elif init == "kaiming_uniform":
                bound = math.sqrt(6.0 / fi)
                p.uniform_(-bound, bound, generator=generator)
            else:
                std = math.sqrt(2.0 / fi)
                if role == "Wb" and spec.family in ("t4", "t2and4", "proposed"):
                    std *= 0.1
                p.normal_(0.0, std, generator=generator)


class _QuadBase(nn.Module):
    def __init__(self, spec, compute_dtype=torch.bfloat16, init="reference", device=None,
                 generator=None, recompute_ab=False):
        super().__init__()
        validate_device_spec(spec)
        self.spec = spec
        self.compute_dtype = compute_dtype
        # retain only x between forward and backward; a, b are rebuilt in the backward
        self.recompute_ab = recompute_ab
        for role, shape in param_shapes(spec).items():
            self.register_parameter(role, nn.Parameter(
                torch.empty(shape, dtype=torch.float32, device=device)))
        _reset(self, spec, generator, init)

    def params(self):
        return {role: getattr(self, role) for role in param_shapes(self.spec)}

    def compute_opts(self):
        """the dtype argument of the autograd functions: (dtype, recompute) when recomputing"""
        return (self.compute_dtype, True) if self.recompute_ab else self.compute_dtype

    def forward(self, x):
        roles = tuple(param_shapes(self.spec).keys())
        return QuadFunction.apply(self.spec, self.compute_opts(), x,
                                  *[getattr(self, r) for r in roles])

    def extra_repr(self):
        return self.spec.describe() + f" dtype={self.compute_dtype}"


class QuadConv2d(_QuadBase):
    """Quadratic conv: family in {proposed, t4, t2, t2_linear, first_order}."""

    def __init__(self, in_channels, out_channels, kernel_size=3, stride=1, padding=0,
                 family="proposed", compute_dtype=torch.bfloat16, init="reference",
                 device=None, generator=None):
        spec = QuadraticLayerSpec(kind="conv", family=family, in_dim=in_channels,
                                  out_dim=out_channels, kernel=kernel_size, stride=stride,
                                  pad=padding)
        super().__init__(spec, compute_dtype, init, device, generator)


class QuadLinear(_QuadBase):
    """Quadratic fc layer; weights stored (in, out) like the reference."""

    def __init__(self, in_features, out_features, family="proposed",
                 compute_dtype=torch.bfloat16, init="reference", device=None, generator=None):
        spec = QuadraticLayerSpec(kind="fc", family=family, in_dim=in_features,
                                  out_dim=out_features)
        super().__init__(spec, compute_dtype, init, device, generator)
