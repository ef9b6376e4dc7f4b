"""Fused SGD + weight pack.

``QuadSGD`` applies the reference ``sgd_step`` (trainer.py:50-61:
v <- m v + g + wd p, first step v = g + wd p; p <- p - lr v -- the same update
as ``torch.optim.SGD(momentum=m, weight_decay=wd, dampening=0)``) to every
parameter. For the weight roles of the quadratic modules it runs one kernel
per layer (``qd_sgd_pack``) that updates the fp32 masters and momentum in
place AND writes the packed bf16 layouts the forward / backward kernels
consume; the pack is registered on the weights' current versions, so the
next forward skips its own packing launch. Gradients are read where autograd
(or the data-parallel buckets of ``dp.BucketedAllReduce``) left them. All
other parameters (biases, first-order layers, BN) go through
``torch.optim.SGD`` with the same hyper-parameters.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib, neurons
from .nn import _QuadBase


def _pack_shape(spec):
    """an input shape for the layer's descriptor: the packed layout does not
    depend on the batch / image size"""
    return (1, spec.in_dim) if spec.kind == "fc" else (1, spec.in_dim, spec.kernel, spec.kernel)


class QuadSGD(torch.optim.Optimizer):
    def __init__(self, model, lr=0.1, momentum=0.9, weight_decay=5e-4):
        # fp32 layers on the split tensor-core path (device path 3) pack their own
        # [hi | lo | hi] layout in the forward: they take the plain SGD below
        self.quad = [m for m in model.modules() if isinstance(m, _QuadBase) and m.spec.kind != "dwconv"
                     and not m.spec.family.startswith("t1") and neurons.device_path(
                         m.spec, _pack_shape(m.spec), m.compute_dtype) != 3]
        fused = set()
        for m in self.quad:
            for r in neurons.WEIGHT_ROLES[m.spec.family]:
                fused.add(id(getattr(m, r)))
        # the kernel indexes weights in the reference layouts ((F, C, r, r) / (in, out)),
        # so a module moved to channels_last gets its quadratic weights back in the
        # standard layout (autograd then also produces gradients in that layout)
        for m in self.quad:
            for r in neurons.WEIGHT_ROLES[m.spec.family]:
                w = getattr(m, r)
                if not w.is_contiguous():
                    w.data = w.data.contiguous()
        # every other parameter too: the gradients the library and the DP buckets
        # produce are in the standard layout, and a channels_last parameter would
        # make autograd accumulate them strided (gradient layout contract)
        for p in model.parameters():
            if not p.is_contiguous():
                p.data = p.data.contiguous()
        params = [p for p in model.parameters() if p.requires_grad]
        defaults = dict(lr=lr, momentum=momentum, weight_decay=weight_decay)
        super().__init__(params, defaults)
        rest = [p for p in params if id(p) not in fused]
        self._rest = torch.optim.SGD(rest, lr=lr, momentum=momentum, weight_decay=weight_decay,
                                     dampening=0.0, foreach=True) if rest else None
        self._packs = {}
        self._streams = []
        self.nstreams = 4  # streams the per-layer update + pack kernels are spread over

    @torch.no_grad()
    def step(self, closure=None):
        loss = closure() if closure is not None else None
        g = self.param_groups[0]
        lr, mom, wd = g["lr"], g["momentum"], g["weight_decay"]
        lib = _lib.load()
        # pass 1 on the current stream: state, packs and descriptors (allocations and
        # first-time packs are ordered on it)
        cur = torch.cuda.current_stream()
        work = []
        for m in self.quad:
            roles = neurons.WEIGHT_ROLES[m.spec.family]
            ws = [getattr(m, r) for r in roles]
            if any(w.grad is None for w in ws):
                continue
            states = [self.state[w] for w in ws]
            first = "momentum_buffer" not in states[0]
            for w, stt in zip(ws, states):
                if "momentum_buffer" not in stt:
                    stt["momentum_buffer"] = torch.zeros_like(w, memory_format=torch.contiguous_format)
            desc = neurons.make_desc(m.spec, _pack_shape(m.spec), m.compute_dtype)
            key = id(m)
            wpack = self._packs.get(key)
            if wpack is None:
                # once: a full pack (it also writes the layout's structural zeros)
                wpack = neurons._pack(m.spec, desc, m.params())[0]
                self._packs[key] = wpack
            if not all(w.is_contiguous() for w in ws):
                raise RuntimeError("QuadSGD: quadratic weights must stay in the standard contiguous layout")
            grads = [w.grad.contiguous() for w in ws]
            work.append((ws, states, first, desc, wpack, grads))
        # pass 2: the per-layer update + pack kernels are independent; spread over a
        # few streams forked from the current one (most layers are small and
        # latency-bound), joined back before the rest of the step
        nstreams = min(self.nstreams, len(work))
        if nstreams > 1:
            if len(self._streams) < nstreams:
                self._streams = [torch.cuda.Stream(device=cur.device) for _ in range(nstreams)]
            for sx in self._streams[:nstreams]:
                sx.wait_stream(cur)
        for li, (ws, states, first, desc, wpack, grads) in enumerate(work):
            stream = (self._streams[li % nstreams] if nstreams > 1 else cur).cuda_stream
            st = lib.qd_sgd_pack(ctypes.byref(desc), _lib.ptr3(*[w.data_ptr() for w in ws]),
                                 _lib.ptr3(*[s_["momentum_buffer"].data_ptr() for s_ in states]),
                                 _lib.ptr3(*[gr.data_ptr() for gr in grads]), float(lr), float(mom),
                                 float(wd), int(first), wpack.data_ptr(), stream)
            _lib.raise_for(st, "qd_sgd_pack")
            for w in ws:  # the kernel changed the weights in place: bump their version counters
                torch.autograd.graph.increment_version(w)
            neurons.register_pack(desc, ws, wpack)
        if nstreams > 1:
            for sx in self._streams[:nstreams]:
                cur.wait_stream(sx)
        if self._rest is not None:
            self._sync_rest()
            self._rest.step()
        return loss

    def _sync_rest(self):
        """The non-fused parameters follow this optimizer's hyper-parameters (an LR
        schedule such as the reference's per-epoch cosine_lr, trainer.py:210,
        edits ``self.param_groups``)."""
        g = self.param_groups[0]
        for rg in self._rest.param_groups:
            for k in ("lr", "momentum", "weight_decay"):
                rg[k] = g[k]

    def state_dict(self):
        sd = super().state_dict()
        if self._rest is not None:
            sd["rest"] = self._rest.state_dict()
        return sd

    def load_state_dict(self, state_dict):
        state_dict = dict(state_dict)
        rest = state_dict.pop("rest", None)
        super().load_state_dict(state_dict)
        if rest is not None and self._rest is not None:
            self._rest.load_state_dict(rest)
        # the packed layouts were written from the old weights: repack on the next step
        self._packs.clear()
