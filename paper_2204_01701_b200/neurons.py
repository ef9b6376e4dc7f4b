"""Drop-in quadratic-layer API on the B200 kernels.

Same names and argument meaning as the reference's ``quadra.neurons``:

* ``forward(spec, params, x) -> (y, LayerCache)``     neurons.py:235-276
* ``symbolic_backward(spec, params, cache, dy) -> (grads, dx)``  neurons.py:295-445
* ``validate_spec``, ``param_shapes``, ``cache_names``, ``count_*``,
  ``init_params``                                        neurons.py:50-186
* ``SYMBOLIC_BACKWARD`` family -> rule registry          tensor.py:598, neurons.py:462-463

Differences a caller sees: tensors are torch tensors on the GPU instead of
``quadra.Tensor`` (numpy inputs and objects with a ``.data`` ndarray are
accepted and moved to the device); arithmetic is fp32 or bf16 instead of
fp64 (``dtype=``, default: x's dtype, fp64 -> fp32); conv activations use the
channels_last memory format (logical NCHW shape is kept). Errors raise the
reference exception classes with the reference messages. Every call runs the
CUDA kernels of libquadra_b200.so; nothing here computes on the CPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import DimensionError, IntegrityError
from .spec import (DEVICE_FAMILIES, FAMILIES, KINDS, QUADRATIC_FAMILIES, T1_FAMILIES,  # noqa: F401
                   QuadraticLayerSpec, cache_names, conv_out_size, count_macs, count_params,
                   count_weights, fan_in, output_spatial, param_shapes, validate_device_spec,
                   validate_spec)

# weight roles in GEMM-branch order and bias roles, per family (the C ABI's
# w[0..2] / bias[0..2] slots)
WEIGHT_ROLES = {"proposed": ("Wa", "Wb", "Wc"), "t4": ("Wa", "Wb"), "t2": ("Wa",), "t3": ("Wa",),
                "first_order": ("W",), "t2_linear": ("Wa", "Wc"), "t2and4": ("Wa", "Wb", "Wc"),
                "t1_pure": ("Wq",), "t1_full": ("Wq", "Wb"), "t1and2": ("Wq", "Wb")}
BIAS_ROLES = {"proposed": ("ba", "bb", "bc"), "first_order": ("b",)}
# gradient dict order of the reference symbolic_backward (neurons.py:380-391, :433-444)
GRAD_ORDER = {"proposed": ("bc", "Wc", "bb", "Wb", "ba", "Wa"), "t4": ("Wb", "Wa"),
              "t2": ("Wa",), "t3": ("Wa",), "first_order": ("b", "W"), "t2_linear": ("Wa", "Wc"),
              "t2and4": ("Wc", "Wb", "Wa"), "t1_pure": ("Wq",), "t1_full": ("Wb", "Wq"),
              "t1and2": ("Wb", "Wq")}

_DAMPED_SECOND_FACTOR = ("t4", "t2and4", "proposed")


@dataclass
class LayerCache:
    """Minimal forward values retained for the closed-form backward.

    Fields of the reference LayerCache (neurons.py:201-209) plus the device
    descriptor and the packed weights the forward used.
    """
    family: str
    kind: str
    x: torch.Tensor
    a: torch.Tensor | None
    b: torch.Tensor | None
    y_shape: tuple
    desc: object = field(default=None, repr=False)
    wpack: torch.Tensor | None = field(default=None, repr=False)
    pack_key: tuple = field(default=(), repr=False)
    # recompute mode: a, b are not retained; the backward
    # rebuilds them from x with the forward kernels
    recompute: bool = field(default=False, repr=False)


def _device():
    if not torch.cuda.is_available():
        from .errors import DeviceError
        raise DeviceError("no CUDA device: the quadratic-layer kernels run only on the GPU")
    return torch.device("cuda", torch.cuda.current_device())


def _as_device(t):
    if isinstance(t, torch.Tensor):
        return t if t.is_cuda else t.to(_device())
    if hasattr(t, "data") and isinstance(getattr(t, "data"), np.ndarray):
        t = t.data
    return torch.as_tensor(np.asarray(t), device=_device())


def _compute_dtype(x, dtype):
    if dtype is not None:
        dt = dtype
    else:
        dt = x.dtype
        if dt == torch.float64:
            dt = torch.float32
    if dt not in (torch.float32, torch.bfloat16):
        raise DimensionError(f"unsupported compute dtype {dt}; use float32 or bfloat16")
    return dt


def _check_x(spec, x):
    """neurons.py:212-220."""
    if spec.kind == "fc":
        if x.ndim != 2 or x.shape[1] != spec.in_dim:
            raise DimensionError(f"layer expects (N, {spec.in_dim}) input, got {tuple(x.shape)}")
    else:
        if x.ndim != 4 or x.shape[1] != spec.in_dim:
            raise DimensionError(
                f"layer expects (N, {spec.in_dim}, H, W) input, got {tuple(x.shape)}")


def make_desc(spec, x_shape, dtype, flags=0):
    d = _lib.QdDesc()
    d.family = _lib.FAMILY_CODE[spec.family]
    d.kind = _lib.KIND_CODE[spec.kind]
    d.dtype = _lib.BF16 if dtype == torch.bfloat16 else _lib.F32
    d.N = int(x_shape[0])
    d.C = int(x_shape[1])
    d.H = int(x_shape[2]) if spec.kind != "fc" else 1
    d.W = int(x_shape[3]) if spec.kind != "fc" else 1
    d.F = spec.out_dim
    d.r, d.stride, d.pad = spec.kernel, spec.stride, spec.pad
    d.flags = flags
    return d


def _layout(t, kind):
    return t.contiguous(memory_format=torch.channels_last) if kind != "fc" else t.contiguous()


def _weights(spec, params):
    shapes = param_shapes(spec)
    out = {}
    for role, shape in shapes.items():
        if role not in params:
            raise DimensionError(f"missing parameter {role!r} for family {spec.family}")
        t = _as_device(params[role])
        if tuple(t.shape) != tuple(shape):
            raise DimensionError(f"parameter {role} has shape {tuple(t.shape)}, expected {shape}")
        out[role] = t
    return out


def _pack_key(ws):
    return tuple((id(t), t._version, t.data_ptr()) for t in ws)


def _pack_tag(desc):
    """layout identity of a packed weight buffer (it does not depend on N, H, W)"""
    return (desc.family, desc.kind, desc.dtype, desc.C, desc.F, desc.r)


def _registered_pack(desc, ws):
    """A packed buffer the fused optimizer (optim.QuadSGD) registered for exactly
    these weight versions, else None. Only that optimizer registers packs, so
    the default path packs on every call as before."""
    hit = getattr(ws[0], "_qd_pack", None)
    if hit is None:
        return None
    tag, key, wpack = hit
    if tag == _pack_tag(desc) and key == _pack_key(ws):
        return wpack
    return None


def register_pack(desc, params_by_role, wpack):
    """Record `wpack` as the packed layout of the current weight versions."""
    ws = list(params_by_role)
    setattr(ws[0], "_qd_pack", (_pack_tag(desc), _pack_key(ws), wpack))


def _pack(spec, desc, params):
    lib = _lib.load()
    roles = WEIGHT_ROLES[spec.family]
    P = _weights(spec, params)
    hit = _registered_pack(desc, [P[r] for r in roles])
    if hit is not None:
        biases = [P[r].detach().to(torch.float32).contiguous() for r in BIAS_ROLES.get(spec.family, ())]
        return hit, _pack_key([P[r] for r in roles]), biases, None
    ws = [P[r].detach().to(torch.float32).contiguous() for r in roles]
    nbytes = lib.qd_pack_bytes(ctypes.byref(desc))
    if nbytes == 0:
        _lib.raise_for(lib.qd_validate(ctypes.byref(desc)), "pack")
    wpack = torch.empty(nbytes, dtype=torch.uint8, device=ws[0].device)
    st = lib.qd_pack_weights(ctypes.byref(desc), _lib.ptr3(*[w.data_ptr() for w in ws]),
                             wpack.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _lib.raise_for(st, "qd_pack_weights")
    biases = [P[r].detach().to(torch.float32).contiguous() for r in BIAS_ROLES.get(spec.family, ())]
    return wpack, _pack_key([P[r] for r in roles]), biases, ws


def _workspace(desc, device):
    n = _lib.load().qd_workspace_bytes(ctypes.byref(desc))
    return torch.empty(max(n, 1), dtype=torch.uint8, device=device)


def split_opts(dtype):
    """A module's compute option: a dtype, or (dtype, recompute_ab)."""
    if isinstance(dtype, tuple):
        return dtype[0], bool(dtype[1])
    return dtype, False


def bn_stats_rows(spec, x_shape, dtype, flags=0):
    """Rows of BN statistics the forward epilogue writes for this layer (0: none;
    the BN that follows then reduces y itself). C ABI qd_bn_stats_rows."""
    desc = make_desc(spec, x_shape, dtype, flags)
    return int(_lib.load().qd_bn_stats_rows(ctypes.byref(desc)))


def forward(spec, params, x, *, dtype=None, flags=0, recompute=False, bn_stats=None):
    """Evaluate one layer on the GPU; returns (y, LayerCache). neurons.py:235-276.

    recompute=True: the cache keeps x only (the a, b buffers the kernels write are
    not retained); the backward rebuilds a, b with one more forward GEMM.
    bn_stats: an fp32 buffer of ``bn_stats_rows * (2 F + 1)`` floats the fprop
    epilogue fills with the BN statistics of y (bn.QuadConvBN)."""
    validate_device_spec(spec)
    lib = _lib.load()
    x = _as_device(x)
    _check_x(spec, x)
    cdt = _compute_dtype(x, dtype)
    x = _layout(x.detach().to(cdt), spec.kind)
    desc = make_desc(spec, x.shape, cdt, flags)
    _lib.raise_for(lib.qd_validate(ctypes.byref(desc)))
    oh, ow = ctypes.c_int(), ctypes.c_int()
    lib.qd_out_shape(ctypes.byref(desc), ctypes.byref(oh), ctypes.byref(ow))
    wpack, key, biases, _ = _pack(spec, desc, params)
    if spec.kind != "fc":
        yshape = (x.shape[0], spec.out_dim, oh.value, ow.value)
        mk = lambda: torch.empty(yshape, dtype=cdt, device=x.device,  # noqa: E731
                                 memory_format=torch.channels_last)
    else:
        yshape = (x.shape[0], spec.out_dim)
        mk = lambda: torch.empty(yshape, dtype=cdt, device=x.device)  # noqa: E731
    y = mk()
    a = b = None
    if spec.family in ("proposed", "t4", "t2and4"):
        a, b = mk(), mk()
    ws = _workspace(desc, x.device)
    if bn_stats is not None:
        st = lib.qd_forward_bnstats(ctypes.byref(desc), x.data_ptr(), wpack.data_ptr(),
                                    _lib.ptr3(*[t.data_ptr() for t in biases]), y.data_ptr(),
                                    a.data_ptr() if a is not None else None,
                                    b.data_ptr() if b is not None else None, ws.data_ptr(), bn_stats.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream)
        _lib.raise_for(st, "qd_forward_bnstats")
    else:
        st = lib.qd_forward(ctypes.byref(desc), x.data_ptr(), wpack.data_ptr(),
                            _lib.ptr3(*[t.data_ptr() for t in biases]), y.data_ptr(),
                            a.data_ptr() if a is not None else None,
                            b.data_ptr() if b is not None else None, ws.data_ptr(),
                            torch.cuda.current_stream().cuda_stream)
        _lib.raise_for(st, "qd_forward")
    if recompute and a is not None:
        return y, LayerCache(spec.family, spec.kind, x, None, None, tuple(y.shape), desc, wpack, key, True)
    return y, LayerCache(spec.family, spec.kind, x, a, b, tuple(y.shape), desc, wpack, key)


def restore_ab(spec, params, cache):
    """Recompute mode: a, b of the cached x through the forward kernels (the
    fused GEMM also recomputes Wc x: +1/3 of the forward GEMM work). Returns
    (a, b) without storing them in the cache, so they die with the backward."""
    if not cache.recompute or cache.a is not None:
        return cache.a, cache.b
    _, c2 = forward(spec, params, cache.x, dtype=cache.x.dtype,
                    flags=cache.desc.flags if cache.desc is not None else 0)
    return c2.a, c2.b


def _grad_buffers(shapes, roles, dev, out):
    """fp32 gradient outputs: ``out[role]`` (a caller-owned contiguous fp32 tensor of
    the role's shape, e.g. a data-parallel bucket view) or a fresh tensor"""
    res = {}
    for r in roles:
        t = (out or {}).get(r)
        if t is None or tuple(t.shape) != tuple(shapes[r]) or t.dtype != torch.float32 or not t.is_contiguous():
            t = torch.empty(shapes[r], dtype=torch.float32, device=dev)
        res[r] = t
    return res


def symbolic_backward(spec, params, cache, dy, *, want_dx=True, want_dw=True, want_db=True, out=None):
    """Closed-form gradients on the GPU; returns ({role: grad}, dx).

    neurons.py:295-445 -- same checks (IntegrityError for a cache of another
    family/kind or a dy of the wrong shape), same roles, reference layouts.
    Weight/bias gradients are fp32; dx has the compute dtype (None when
    want_dx is False).
    """
    if cache.family != spec.family or cache.kind != spec.kind:
        raise IntegrityError(
            f"cache for {cache.family}/{cache.kind} used with {spec.family}/{spec.kind} layer")
    validate_device_spec(spec)
    lib = _lib.load()
    g = _as_device(dy.data if hasattr(dy, "data") and not isinstance(dy, (torch.Tensor, np.ndarray)) else dy)
    if tuple(g.shape) != tuple(cache.y_shape):
        raise IntegrityError(
            f"output gradient shape {tuple(g.shape)} does not match forward {tuple(cache.y_shape)}")
    _check_x(spec, cache.x)
    x = cache.x
    cdt = x.dtype
    g = _layout(g.detach().to(cdt), spec.kind)
    flags = cache.desc.flags if cache.desc is not None else 0
    if not want_dx:
        flags |= _lib.FLAG_NO_DX
    if not want_dw:
        flags |= _lib.FLAG_NO_DW
    desc = make_desc(spec, x.shape, cdt, flags)
    P = _weights(spec, params)
    roles = WEIGHT_ROLES[spec.family]
    if cache.wpack is not None and cache.pack_key == _pack_key([P[r] for r in roles]):
        wpack = cache.wpack
    else:
        wpack = _pack(spec, desc, params)[0]
    dev = x.device
    shapes = param_shapes(spec)
    broles = BIAS_ROLES.get(spec.family, ()) if want_db else ()  # want_db=False: no bias grads (constant bias)
    grads = _grad_buffers(shapes, [role for role in GRAD_ORDER[spec.family]
                                   if want_db or role not in BIAS_ROLES.get(spec.family, ())], dev, out)
    dx = torch.empty_like(x) if want_dx else None  # preserves channels_last
    ws = _workspace(desc, dev)
    ca, cb = restore_ab(spec, params, cache)
    st = lib.qd_backward(ctypes.byref(desc), x.data_ptr(), wpack.data_ptr(),
                         ca.data_ptr() if ca is not None else None,
                         cb.data_ptr() if cb is not None else None,
                         g.data_ptr(), dx.data_ptr() if dx is not None else None,
                         _lib.ptr3(*[grads[r].data_ptr() for r in roles]),
                         _lib.ptr3(*[grads[r].data_ptr() for r in broles]),
                         ws.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _lib.raise_for(st, "qd_backward")
    return grads, dx


def backward_from_D(spec, params, cache, D, *, want_dx=True, want_dw=True, out=None):
    """Layer backward from a precomputed operand D ([M, Jd] rows, e.g. from the
    fused BN backward ``bn.bn_backward_D``); weight gradients and dx only (the
    bias gradients come with D). Stride-1 fc / conv layers."""
    lib = _lib.load()
    x = cache.x
    cdt = x.dtype
    flags = (cache.desc.flags if cache.desc is not None else 0) | _lib.FLAG_D_GIVEN
    if not want_dx:
        flags |= _lib.FLAG_NO_DX
    if not want_dw:
        flags |= _lib.FLAG_NO_DW
    desc = make_desc(spec, x.shape, cdt, flags)
    P = _weights(spec, params)
    roles = WEIGHT_ROLES[spec.family]
    if cache.wpack is not None and cache.pack_key == _pack_key([P[r] for r in roles]):
        wpack = cache.wpack
    else:
        wpack = _pack(spec, desc, params)[0]
    dev = x.device
    shapes = param_shapes(spec)
    grads = _grad_buffers(shapes, roles, dev, out)
    dx = torch.empty_like(x) if want_dx else None
    ws = _workspace(desc, dev)
    st = lib.qd_backward(ctypes.byref(desc), x.data_ptr(), wpack.data_ptr(), None, None, D.data_ptr(),
                         dx.data_ptr() if dx is not None else None,
                         _lib.ptr3(*[grads[r].data_ptr() for r in roles]), _lib.ptr3(), ws.data_ptr(),
                         torch.cuda.current_stream().cuda_stream)
    _lib.raise_for(st, "qd_backward (D given)")
    return grads, dx


def device_path(spec, x_shape, dtype=torch.bfloat16, flags=0):
    """0 = generic CUDA-core kernels, 1 = tcgen05/TMA kernels (bf16), 2 = depth-wise
    kernels, 3 = fp32 on the tcgen05 kernels through split bf16 operands
    (hi*hi + hi*lo + lo*hi, qd_x3.cu)."""
    desc = make_desc(spec, x_shape, dtype, flags)
    p = _lib.load().qd_path(ctypes.byref(desc))
    if p < 0:
        _lib.raise_for(_lib.load().qd_validate(ctypes.byref(desc)))
    return p


def init_params(spec, rng, device=None):
    """Fan-in-scaled normal init, product second factor damped x0.1, zero biases.

    Same draws, in the same order, as the reference init_params
    (neurons.py:132-147) given the same numpy Generator; returns fp32 torch
    tensors on the GPU.
    """
    shapes = param_shapes(spec)
    std = np.sqrt(2.0 / fan_in(spec))
    dev = device or _device()
    out = {}
    for role, shape in shapes.items():
        if role.startswith("b"):
            arr = np.zeros(shape)
        elif role == "Wq":
            arr = rng.normal(0.0, 1.0 / spec.in_dim, size=shape)
        elif role == "Wb" and spec.family in _DAMPED_SECOND_FACTOR:
            arr = rng.normal(0.0, 0.1 * std, size=shape)
        else:
            arr = rng.normal(0.0, std, size=shape)
        out[role] = torch.as_tensor(arr, dtype=torch.float32, device=dev)
    return out


# ---------------------------------------------------------------------------
# tape / plugin-registry boundary (reference neurons.py:448-477, tensor.py:598-609)
# ---------------------------------------------------------------------------
SYMBOLIC = "symbolic"  # reference tensor.py:31 (tape mode of a closed-form node)

_dev_ids = __import__("itertools").count(1 << 40)  # ids of device-tensor wrappers


class DeviceTensor:
    """Tape-facing wrapper of a device tensor for tapes whose inputs are torch
    tensors: the attributes the reference Tape reads (``id``, ``shape``,
    ``nbytes``, ``is_param``; tensor.py:43-90, :151-185) over ``data``."""

    __slots__ = ("data", "id", "is_param")

    def __init__(self, data, is_param=False):
        self.data = data
        self.id = next(_dev_ids)
        self.is_param = is_param

    @property
    def shape(self):
        return tuple(self.data.shape)

    @property
    def nbytes(self):
        return self.data.numel() * self.data.element_size()


def _host_array(t):
    """device tensor -> C-contiguous fp64 ndarray (the reference's array type)."""
    return np.ascontiguousarray(t.detach().to(torch.float64).cpu().numpy())


def _wrap_like(x, t):
    """Result tensor of the caller's kind: a reference ``Tensor`` (fp64 host
    copy, via the class's own ``_wrap``) when x is one, else a DeviceTensor."""
    if t is None:
        return None
    if isinstance(x, torch.Tensor) or not hasattr(type(x), "_wrap"):
        return DeviceTensor(t)
    return type(x)._wrap(_host_array(t))


def record_symbolic(tape, spec, params, x, tag="", *, dtype=None):
    """Run a layer forward on the GPU and record it on ``tape`` as ONE symbolic
    node retaining ``cache_names(family)`` (reference neurons.py:466-477).

    ``tape`` is any object with the reference ``Tape.record(op, arrays,
    input_names, tag=, mode=, meta=)`` method (tensor.py:151); ``x`` a reference
    ``Tensor`` (fp64, host) or a torch tensor. The node's arrays are the
    caller's tensor kind (the reference tape accounts their bytes); the device
    cache rides along in ``meta["b200_cache"]`` so the registered backward
    (``_quad_node_backward``) runs from the device-resident x, a, b.
    """
    xin = x.data if (not isinstance(x, torch.Tensor) and hasattr(x, "data")) else x
    y, cache = forward(spec, params, xin, dtype=dtype)
    yt = _wrap_like(x, y)
    xt = x if not isinstance(x, torch.Tensor) else DeviceTensor(x)
    arrays = {"out": yt, "x": xt}
    if cache.a is not None:
        arrays["a"] = _wrap_like(x, cache.a)
        arrays["b"] = _wrap_like(x, cache.b)
    tape.record("quad", arrays, ("x",), tag=tag, mode=SYMBOLIC,
                meta={"family": spec.family, "spec": spec, "params": params,
                      "retain": cache_names(spec.family), "b200_cache": cache})
    return yt


def _node_cache(node, spec):
    """The device LayerCache of a tape node: the one record_symbolic stored, or
    (a node the reference recorded itself) one rebuilt from the node's arrays."""
    cache = node.meta.get("b200_cache")
    if cache is not None:
        return cache
    x = node.arrays["x"]
    xa = _as_device(x.data if hasattr(x, "data") and not isinstance(x, torch.Tensor) else x)
    _check_x(spec, xa)
    cdt = _compute_dtype(xa, None)
    xa = _layout(xa.detach().to(cdt), spec.kind)

    def dev(name):
        t = node.arrays.get(name)
        if t is None:
            return None
        t = _as_device(t.data if hasattr(t, "data") and not isinstance(t, torch.Tensor) else t)
        return _layout(t.detach().to(cdt), spec.kind)
    return LayerCache(spec.family, spec.kind, xa, dev("a"), dev("b"), tuple(node.arrays["out"].shape),
                      make_desc(spec, xa.shape, cdt))


def _quad_node_backward(node, g):
    """Registry contract ``fn(node, g) -> [(tensor_id, grad), ...]`` of the
    reference (tensor.py:598-609; adapter neurons.py:448-459): the closed-form
    backward of one symbolic quadratic node, computed on the GPU.

    Gradients come back in the kind of ``g``: fp64 ndarrays when the tape is
    the reference's (its sweep adds them with numpy, tensor.py:634-637), torch
    tensors otherwise.
    """
    spec = node.meta["spec"]
    params = node.meta["params"]
    cache = _node_cache(node, spec)
    host = not isinstance(g, torch.Tensor)
    gin = g.data if (host and hasattr(g, "data") and not isinstance(g, np.ndarray)) else g
    grads, dx = symbolic_backward(spec, params, cache, gin)
    conv = _host_array if host else (lambda t: t)
    out = [(node.arrays["x"].id, conv(dx))]
    for role, grad in grads.items():
        p = params[role]
        out.append((p.id if hasattr(p, "id") else id(p), conv(grad)))
    return out


# family -> closed-form backward rule with the registry contract fn(node, g)
# (reference tensor.py:598, populated at import like neurons.py:462-463)
SYMBOLIC_BACKWARD = {fam: _quad_node_backward for fam in DEVICE_FAMILIES}


def install(tensor_module, families=None):
    """Route a reference tape's quadratic nodes to the device: register
    ``_quad_node_backward`` in the reference's ``tensor.SYMBOLIC_BACKWARD``
    (tensor.py:598) for ``families`` (default: every family both support).
    Returns the previous entries so a caller can restore them."""
    reg = tensor_module.SYMBOLIC_BACKWARD
    fams = families or [f for f in reg if f in DEVICE_FAMILIES]
    prev = {f: reg.get(f) for f in fams}
    for f in fams:
        reg[f] = _quad_node_backward
    return prev


def uninstall(tensor_module, prev):
    """Restore the registry entries ``install`` returned."""
    reg = tensor_module.SYMBOLIC_BACKWARD
    for f, fn in prev.items():
        if fn is None:
            reg.pop(f, None)
        else:
            reg[f] = fn
