"""Batch norm (+ ReLU) fused around the quadratic conv.

Reference semantics (tensor.py:423-470 forward, :552-570 backward): batch
statistics over (N, H, W) with the *biased* variance, used both to normalise
and to update the running variance (momentum 0.1, eps 1e-5); eval mode uses
the running statistics.

``QuadConvBN`` = quadratic layer -> BN -> optional ReLU as ONE autograd node:

* forward: the layer kernels produce y (and the a, b cache), one reduction
  pass forms the batch statistics, one pass writes relu(BN(y));
* backward: one reduction pass over (dz, y) gives dgamma / dbeta, ONE
  elementwise pass applies the BN (+ReLU) backward and directly emits the
  layer's backward operand D = [dy b | dy a | dy] and its bias gradients,
  then the layer's wgrad / dgrad kernels run from D (``QD_FLAG_D_GIVEN``).
  The BN-backward output dy is never materialised.

Layers the fused backward does not cover (stride 2 off the direct path, t3,
T1 families, dwconv)
use the same reference BN semantics through torch ops (autograd).
"""

from __future__ import annotations

import ctypes
import os

import torch
from torch import nn

from . import _lib, neurons
from .nn import QuadFunction, _QuadBase, grad_sinks, settle_sinks
from .spec import QuadraticLayerSpec, param_shapes


def _rows(t):
    """[M, C] row view of an NHWC (channels_last) or 2-D tensor (no copy)."""
    if t.dim() == 4:
        n, c, h, w = t.shape
        return t.permute(0, 2, 3, 1).reshape(n * h * w, c)
    return t


def _dtype_code(t):
    return _lib.BF16 if t.dtype == torch.bfloat16 else _lib.F32


def bn_forward(y, gamma, beta, running_mean, running_var, momentum, eps, relu, training, res=None):
    """z = relu?(gamma (y - mean) inv_std + beta [+ res]); returns (z, save_mean, save_invstd)."""
    lib = _lib.load()
    yr = _rows(y)
    M, C = yr.shape
    if not yr.is_contiguous():
        raise ValueError("bn_forward expects channels_last / row-major input")
    z = torch.empty_like(y)
    if training:
        sm = torch.empty(C, dtype=torch.float32, device=y.device)
        si = torch.empty(C, dtype=torch.float32, device=y.device)
    else:
        sm = running_mean.float().contiguous()
        si = torch.rsqrt(running_var.float() + eps).contiguous()
    ws = torch.empty(lib.qd_bn_workspace_bytes(M, C, C), dtype=torch.uint8, device=y.device)
    if res is None:
        st = lib.qd_bn_forward(M, C, _dtype_code(y), y.data_ptr(), gamma.data_ptr(), beta.data_ptr(),
                               running_mean.data_ptr() if training else None,
                               running_var.data_ptr() if training else None, float(momentum), float(eps),
                               int(relu), int(training), z.data_ptr(), sm.data_ptr(), si.data_ptr(), ws.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    else:
        if res.shape != y.shape or res.dtype != y.dtype or not _rows(res).is_contiguous():
            raise ValueError("bn_forward: residual must match y (shape, dtype, channels_last)")
        st = lib.qd_bn_forward_res(M, C, _dtype_code(y), y.data_ptr(), res.data_ptr(), gamma.data_ptr(),
                                   beta.data_ptr(), running_mean.data_ptr() if training else None,
                                   running_var.data_ptr() if training else None, float(momentum), float(eps),
                                   int(relu), int(training), z.data_ptr(), sm.data_ptr(), si.data_ptr(),
                                   ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _lib.raise_for(st, "qd_bn_forward")
    return z, sm, si


def _epilogue_stat_rows(spec, x, dtype):
    """rows of BN statistics the layer's fprop epilogue can write (0: reduce y
    separately). Opt-in (QD_BN_EPI=1): measured slower on the nets (ResNet-18
    13.5k vs 15.6k img/s: the per-warp reductions lengthen the fprop epilogue by
    ~16% and the row merge is latency-bound), DESIGN.md §9."""
    if os.environ.get("QD_BN_EPI", "0") != "1" or x.device.type != "cuda":
        return 0
    dt = dtype if dtype is not None else (torch.float32 if x.dtype == torch.float64 else x.dtype)
    return neurons.bn_stats_rows(spec, tuple(x.shape), dt)


def bn_forward_from_stats(y, stats, rows, gamma, beta, running_mean, running_var, momentum, eps, relu, res=None):
    """BN forward from the fprop epilogue's statistics rows: merge + apply, no
    reduction pass over y. Returns (z, save_mean, save_invstd)."""
    lib = _lib.load()
    yr = _rows(y)
    M, C = yr.shape
    z = torch.empty_like(y)
    sm = torch.empty(C, dtype=torch.float32, device=y.device)
    si = torch.empty(C, dtype=torch.float32, device=y.device)
    if res is not None and (res.shape != y.shape or res.dtype != y.dtype or not _rows(res).is_contiguous()):
        raise ValueError("bn_forward_from_stats: residual must match y (shape, dtype, channels_last)")
    st = lib.qd_bn_forward_stats(M, C, _dtype_code(y), y.data_ptr(), res.data_ptr() if res is not None else None,
                                 stats.data_ptr(), int(rows), gamma.data_ptr(), beta.data_ptr(),
                                 running_mean.data_ptr(), running_var.data_ptr(), float(momentum), float(eps),
                                 int(relu), 1, z.data_ptr(), sm.data_ptr(), si.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream)
    _lib.raise_for(st, "qd_bn_forward_stats")
    return z, sm, si


def _forward_with_stats(spec, params, x, dtype, recompute):
    """layer forward; with the BN statistics rows when its epilogue has them"""
    rows = _epilogue_stat_rows(spec, x, dtype)
    if not rows:
        y, cache = neurons.forward(spec, params, x, dtype=dtype, recompute=recompute)
        return y, cache, None, 0
    stats = torch.empty(rows * (2 * spec.out_dim + 1), dtype=torch.float32, device=x.device)
    y, cache = neurons.forward(spec, params, x, dtype=dtype, recompute=recompute, bn_stats=stats)
    return y, cache, stats, rows


def _f32(C, dev, t=None):
    """a caller-owned fp32 (C,) output (e.g. a data-parallel bucket view) or a fresh one"""
    if t is not None and tuple(t.shape) == (C,) and t.dtype == torch.float32 and t.is_contiguous():
        return t
    return torch.empty(C, dtype=torch.float32, device=dev)


def bn_backward_D(spec, cache, dz, y, gamma, beta, save_mean, save_invstd, relu, params=None, out=None):
    """(D, dgamma, dbeta, {bias role: grad}) for the layer's backward from D;
    ``out`` may hold caller-owned outputs for "gamma", "beta" and the bias roles."""
    lib = _lib.load()
    desc = neurons.make_desc(spec, cache.x.shape, cache.x.dtype)
    pl = lib  # noqa: F841
    fam = spec.family
    nblk = 3 if fam in ("proposed", "t2and4") else (2 if fam == "t4" else 1)
    C = spec.out_dim
    yr = _rows(y)
    M = yr.shape[0]
    D = torch.empty((M, nblk * C), dtype=y.dtype, device=y.device)
    out = out or {}
    dgamma = _f32(C, y.device, out.get("gamma"))
    dbeta = _f32(C, y.device, out.get("beta"))
    broles = neurons.BIAS_ROLES.get(fam, ())
    db = {r: _f32(C, y.device, out.get(r)) for r in broles}
    ws = torch.empty(lib.qd_bn_workspace_bytes(M, C, nblk * C), dtype=torch.uint8, device=y.device)
    dzr = _rows(dz.contiguous(memory_format=torch.channels_last) if dz.dim() == 4 else dz.contiguous())
    ca, cb = (cache.a, cache.b) if params is None else neurons.restore_ab(spec, params, cache)
    st = lib.qd_bn_backward_D(ctypes.byref(desc), dzr.data_ptr(), y.data_ptr(),
                              ca.data_ptr() if ca is not None else None,
                              cb.data_ptr() if cb is not None else None, gamma.data_ptr(),
                              beta.data_ptr(), save_mean.data_ptr(), save_invstd.data_ptr(), int(relu),
                              D.data_ptr(), dgamma.data_ptr(), dbeta.data_ptr(),
                              _lib.ptr3(*[db[r].data_ptr() for r in broles]), ws.data_ptr(),
                              torch.cuda.current_stream().cuda_stream)
    _lib.raise_for(st, "qd_bn_backward_D")
    return D, dgamma, dbeta, db


class _QuadBNFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, spec, dtype, relu, bn, x, gamma, beta, *tensors):
        roles = tuple(param_shapes(spec).keys())
        params = dict(zip(roles, tensors))
        dtype, recompute = neurons.split_opts(dtype)
        y, cache, stats, rows = _forward_with_stats(spec, params, x, dtype, recompute)
        if stats is not None:
            z, sm, si = bn_forward_from_stats(y, stats, rows, gamma, beta, bn.running_mean, bn.running_var,
                                              bn.momentum, bn.eps, relu)
        else:
            z, sm, si = bn_forward(y, gamma, beta, bn.running_mean, bn.running_var, bn.momentum, bn.eps, relu, True)
        ctx.spec, ctx.roles, ctx.params, ctx.cache, ctx.relu = spec, roles, params, cache, relu
        ctx.gamma, ctx.beta = gamma, beta  # the parameters themselves (gradient sinks)
        ctx.x_dtype = x.dtype
        ctx.save_for_backward(y, gamma, beta, sm, si)
        return z

    @staticmethod
    def backward(ctx, dz):
        y, gamma, beta, sm, si = ctx.saved_tensors
        named = dict(ctx.params, gamma=ctx.gamma, beta=ctx.beta)
        needs = dict({r: ctx.needs_input_grad[7 + i] for i, r in enumerate(ctx.roles)},
                     gamma=ctx.needs_input_grad[5], beta=ctx.needs_input_grad[6])
        sinks = grad_sinks(named, needs)
        D, dgamma, dbeta, db = bn_backward_D(ctx.spec, ctx.cache, dz, y, gamma, beta, sm, si, ctx.relu, ctx.params,
                                             out=sinks)
        want_dx = ctx.needs_input_grad[4]
        grads, dx = neurons.backward_from_D(ctx.spec, ctx.params, ctx.cache, D, want_dx=want_dx, out=sinks)
        grads.update(db)
        grads.update(gamma=dgamma, beta=dbeta)
        grads = settle_sinks(named, sinks, grads)
        if dx is not None and dx.dtype != ctx.x_dtype:
            dx = dx.to(ctx.x_dtype)
        ctx.cache = None
        return (None, None, None, None, dx, grads["gamma"], grads["beta"]) + tuple(grads[r] for r in ctx.roles)


class _QuadBNAddReLUFunction(torch.autograd.Function):
    """quadratic layer -> BN -> + residual -> ReLU (a ResNet block tail) as ONE
    node: the residual add and the ReLU ride on the BN apply pass
    (qd_bn_forward_res). Backward: g = dz masked by z > 0 (one pass; it is also
    the residual's gradient), then the BN backward without ReLU emits the
    layer's D from g as in _QuadBNFunction."""

    @staticmethod
    def forward(ctx, spec, dtype, bn, x, res, gamma, beta, *tensors):
        roles = tuple(param_shapes(spec).keys())
        params = dict(zip(roles, tensors))
        dtype, recompute = neurons.split_opts(dtype)
        y, cache, stats, rows = _forward_with_stats(spec, params, x, dtype, recompute)
        if res.dtype != y.dtype or (y.dim() == 4 and not res.is_contiguous(memory_format=torch.channels_last)):
            res = res.to(y.dtype).contiguous(memory_format=torch.channels_last)
        if stats is not None:
            z, sm, si = bn_forward_from_stats(y, stats, rows, gamma, beta, bn.running_mean, bn.running_var,
                                              bn.momentum, bn.eps, True, res=res)
        else:
            z, sm, si = bn_forward(y, gamma, beta, bn.running_mean, bn.running_var, bn.momentum, bn.eps, True, True,
                                   res=res)
        ctx.spec, ctx.roles, ctx.params, ctx.cache = spec, roles, params, cache
        ctx.gamma, ctx.beta = gamma, beta
        ctx.x_dtype, ctx.res_dtype = x.dtype, res.dtype
        ctx.save_for_backward(y, z, gamma, beta, sm, si)
        return z

    @staticmethod
    def backward(ctx, dz):
        y, z, gamma, beta, sm, si = ctx.saved_tensors
        g = torch.ops.aten.threshold_backward(dz.to(z.dtype), z, 0)
        named = dict(ctx.params, gamma=ctx.gamma, beta=ctx.beta)
        needs = dict({r: ctx.needs_input_grad[7 + i] for i, r in enumerate(ctx.roles)},
                     gamma=ctx.needs_input_grad[5], beta=ctx.needs_input_grad[6])
        sinks = grad_sinks(named, needs)
        D, dgamma, dbeta, db = bn_backward_D(ctx.spec, ctx.cache, g, y, gamma, beta, sm, si, False, ctx.params,
                                             out=sinks)
        want_dx = ctx.needs_input_grad[3]
        grads, dx = neurons.backward_from_D(ctx.spec, ctx.params, ctx.cache, D, want_dx=want_dx, out=sinks)
        grads.update(db)
        grads.update(gamma=dgamma, beta=dbeta)
        grads = settle_sinks(named, sinks, grads)
        if dx is not None and dx.dtype != ctx.x_dtype:
            dx = dx.to(ctx.x_dtype)
        ctx.cache = None
        dres = g if ctx.needs_input_grad[4] else None
        return (None, None, None, dx, dres, grads["gamma"], grads["beta"]) + tuple(grads[r] for r in ctx.roles)


class _BNFunction(torch.autograd.Function):
    """BN (+ReLU) alone on the same kernels (layers the fused backward does not
    cover): the backward's D is the BN input gradient itself (one block)."""

    @staticmethod
    def forward(ctx, y, gamma, beta, bn, relu):
        z, sm, si = bn_forward(y, gamma, beta, bn.running_mean, bn.running_var, bn.momentum, bn.eps, relu, True)
        ctx.relu = relu
        ctx.gamma, ctx.beta = gamma, beta
        ctx.save_for_backward(y, gamma, beta, sm, si)
        return z

    @staticmethod
    def backward(ctx, dz):
        y, gamma, beta, sm, si = ctx.saved_tensors
        dy, dgamma, dbeta = _bn_backward_only(y, dz, gamma, beta, sm, si, ctx.relu,
                                              {"gamma": ctx.gamma, "beta": ctx.beta},
                                              {"gamma": ctx.needs_input_grad[1], "beta": ctx.needs_input_grad[2]})
        return dy, dgamma, dbeta, None, None


def _bn_backward_only(y, dz, gamma, beta, sm, si, relu, named, needs):
    """dL/dy, dgamma, dbeta of a BN (+ReLU) from dz (the mask recomputed from y);
    gamma / beta gradients sunk into their data-parallel buckets when allowed"""
    lib = _lib.load()
    yr = _rows(y)
    M, C = yr.shape
    desc = _lib.QdDesc()
    desc.family, desc.kind = _lib.FAMILY_CODE["first_order"], _lib.KIND_CODE["fc"]
    desc.dtype = _dtype_code(y)
    desc.N, desc.C, desc.H, desc.W, desc.F = M, C, 1, 1, C
    desc.r, desc.stride, desc.pad, desc.flags = 1, 1, 0, 0
    dy = torch.empty_like(y)
    sinks = grad_sinks(named, needs)
    dgamma = _f32(C, y.device, sinks.get("gamma"))
    dbeta = _f32(C, y.device, sinks.get("beta"))
    ws = torch.empty(lib.qd_bn_workspace_bytes(M, C, C), dtype=torch.uint8, device=y.device)
    dzr = _rows(dz.contiguous(memory_format=torch.channels_last) if dz.dim() == 4 else dz.contiguous())
    st = lib.qd_bn_backward_D(ctypes.byref(desc), dzr.data_ptr(), y.data_ptr(), None, None, gamma.data_ptr(),
                              beta.data_ptr(), sm.data_ptr(), si.data_ptr(), int(relu), dy.data_ptr(),
                              dgamma.data_ptr(), dbeta.data_ptr(), _lib.ptr3(), ws.data_ptr(),
                              torch.cuda.current_stream().cuda_stream)
    _lib.raise_for(st, "qd_bn_backward_D (bn only)")
    gr = settle_sinks(named, sinks, {"gamma": dgamma, "beta": dbeta})
    return dy, gr["gamma"], gr["beta"]


def _ref_batchnorm(y, gamma, beta, running_mean, running_var, momentum, eps, training):
    """tensor.py:423-470 with torch ops (autograd) -- the unfused fallback."""
    yf = y.float()
    axes = (0,) if y.dim() == 2 else (0, 2, 3)
    shape = (1, -1) if y.dim() == 2 else (1, -1, 1, 1)
    if training:
        mean = yf.mean(dim=axes)
        var = yf.var(dim=axes, unbiased=False)
        with torch.no_grad():
            running_mean.mul_(1.0 - momentum).add_(momentum * mean.detach())
            running_var.mul_(1.0 - momentum).add_(momentum * var.detach())
    else:
        mean, var = running_mean, running_var
    inv = torch.rsqrt(var + eps)
    return (gamma.view(shape) * (yf - mean.view(shape)) * inv.view(shape) + beta.view(shape)).to(y.dtype)


class _BNState(nn.Module):
    def __init__(self, c, momentum=0.1, eps=1e-5, device=None):
        super().__init__()
        self.momentum, self.eps = momentum, eps
        self.register_buffer("running_mean", torch.zeros(c, device=device))
        self.register_buffer("running_var", torch.ones(c, device=device))


class QuadConvBN(nn.Module):
    """Quadratic conv (or fc) -> batch norm (reference semantics) -> optional ReLU."""

    def __init__(self, layer: _QuadBase, relu=True, momentum=0.1, eps=1e-5):
        super().__init__()
        self.layer = layer
        self.relu = relu
        c = layer.spec.out_dim
        dev = next(layer.parameters()).device
        self.weight = nn.Parameter(torch.ones(c, device=dev))
        self.bias = nn.Parameter(torch.zeros(c, device=dev))
        self.bn = _BNState(c, momentum, eps, dev)

    def fused(self, x=None):
        sp = self.layer.spec
        if os.environ.get("QD_NO_BNFUSE"):
            return False
        if sp.stride == 2:
            # stride 2 fuses when the layer runs on its own output grid (the
            # library's tc_s2_direct: tcgen05 path, plain-K family), so
            # the emitted D is the operand its backward consumes as is
            if x is None or sp.kind != "conv" or sp.family not in ("proposed", "t4", "first_order"):
                return False
            oh = (x.shape[2] + 2 * sp.pad - sp.kernel) // 2 + 1
            ow = (x.shape[3] + 2 * sp.pad - sp.kernel) // 2 + 1
            return (oh <= 128 and ow <= 128 and self.layer.compute_dtype == torch.bfloat16
                    and neurons.device_path(sp, tuple(x.shape), torch.bfloat16) == 1)
        return (sp.stride == 1 and sp.kind in ("conv", "fc") and sp.family not in ("t3", "t1_pure", "t1_full",
                                                                                   "t1and2"))

    def forward_add_relu(self, x, res):
        """relu(BN(layer(x)) + res) -- the block tail of a residual net; one
        fused node on the library kernels when the layer's BN is fused, else the
        composition (the module's own relu flag is not applied here). Reached as
        ``module(x, res)`` (so module hooks see it)."""
        if (self.training and x.device.type == "cuda" and self.fused(x)
                and res.shape[1] == self.layer.spec.out_dim):
            spec = self.layer.spec
            tensors = [getattr(self.layer, r) for r in param_shapes(spec).keys()]
            return _QuadBNAddReLUFunction.apply(spec, self.layer.compute_opts(), self.bn, x, res, self.weight,
                                                self.bias, *tensors)
        relu, self.relu = self.relu, False
        try:
            out = self.forward(x)
        finally:
            self.relu = relu
        return torch.relu(out + res)

    def forward(self, x, res=None):
        if res is not None:
            return self.forward_add_relu(x, res)
        spec = self.layer.spec
        roles = tuple(param_shapes(spec).keys())
        tensors = [getattr(self.layer, r) for r in roles]
        if self.training and self.fused(x):
            return _QuadBNFunction.apply(spec, self.layer.compute_opts(), self.relu, self.bn, x, self.weight,
                                         self.bias, *tensors)
        y = QuadFunction.apply(spec, self.layer.compute_opts(), x, *tensors)
        if self.training and (y.dim() == 2 or y.is_contiguous(memory_format=torch.channels_last)):
            return _BNFunction.apply(y, self.weight, self.bias, self.bn, self.relu)
        z = _ref_batchnorm(y, self.weight, self.bias, self.bn.running_mean, self.bn.running_var, self.bn.momentum,
                           self.bn.eps, self.training)
        return torch.relu(z) if self.relu else z


class BNAct2d(nn.BatchNorm2d):
    """nn.BatchNorm2d (+ fused ReLU) on the library's BN kernels, for the
    first-order parts of the QuadraNets (ResNet stem, downsample shortcuts).

    Same parameters, buffers and state-dict keys as nn.BatchNorm2d; statistics
    follow the reference (tensor.py:423-470): biased batch variance, also in the
    running update. CUDA channels_last / 2-D inputs run ``_BNFunction``; other
    devices (CPU inspection, meta-device FLOP counting) use the torch ops with
    the same semantics."""

    def __init__(self, num_features, relu=False, eps=1e-5, momentum=0.1, device=None, dtype=None):
        super().__init__(num_features, eps=eps, momentum=momentum, device=device, dtype=dtype)
        self.relu = bool(relu)

    def forward(self, x):
        if self.training:
            self.num_batches_tracked.add_(1)
        if x.device.type == "cuda" and (x.dim() == 2 or x.is_contiguous(memory_format=torch.channels_last)):
            if self.training:
                return _BNFunction.apply(x, self.weight, self.bias, self, self.relu)
            # eval: running statistics through the same apply kernel
            z, _, _ = bn_forward(x, self.weight, self.bias, self.running_mean, self.running_var, self.momentum,
                                 self.eps, self.relu, False)
            return z
        z = _ref_batchnorm(x, self.weight, self.bias, self.running_mean, self.running_var, self.momentum, self.eps,
                           self.training)
        return torch.relu(z) if self.relu else z
