"""Data-parallel gradient exchange: bucketed all-reduce overlapped with backward.

The quadratic layer is per-sample independent; the only cross-sample
coupling of batch-sharded training is the sum over samples inside dW / db
(SURVEY.md §8(e)). Each rank runs its own batch and the gradients are
averaged over ranks once per step -- one exchange, no other collective.

Mechanics (one process per GPU, torch.distributed over NCCL on NVLink /
NVSwitch; gloo on CPU for the tests):

* parameters are grouped into flat fp32 buckets (~25 MB) in reverse
  registration order, i.e. roughly the order backward produces them;
* each parameter's ``.grad`` is a view into its bucket, so autograd
  accumulates straight into the bucket (no copy);
* a post-accumulate-grad hook counts ready parameters; when a bucket is
  complete its all-reduce (ReduceOp.AVG) is launched asynchronously, so the
  NCCL transfer of the deep layers overlaps the backward of the shallow ones;
* ``finish()`` waits for the outstanding buckets before the optimizer step.

Direct gradient sink: the library's backward kernels (quadratic layers, their
BN, first-order BN) fold their weight / bias gradients straight into the
bucket views (``take_grad``) instead of fresh tensors, and the autograd
function returns None for those parameters -- no AccumulateGrad add pass
over the ~135 MB of gradients (ResNet-18) per step; the function then marks
the parameter ready (``grad_ready``), which is what the post-accumulate hook
does for every other parameter. A parameter is taken at most once between
``reset()`` calls (a second gradient in the same step accumulates as usual).

The update itself is the reference's ``sgd_step`` (trainer.py:50-61:
v <- m v + g + wd p; p <- p - lr v), which is exactly
``torch.optim.SGD(momentum=0.9, weight_decay=5e-4, dampening=0)``.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


import os as _os

_DEBUG = bool(_os.environ.get("QD_DP_DEBUG"))


def take_grad(p):
    """The tensor a library backward may overwrite with ``p``'s gradient this step
    (its bucket view), or None (then the gradient goes through autograd)."""
    red = getattr(p, "_qd_red", None)
    return red.take(p) if red is not None else None


def grad_ready(p):
    """``p``'s gradient is complete in its bucket (after a ``take_grad`` write)."""
    p._qd_red.ready(p)


def _padded(n, align=32):
    """elements a gradient view occupies in its bucket: rounded up to 32 fp32
    (128 B), so every view starts aligned -- the library's folds write dW with
    16-B vector stores and take a scalar fallback otherwise (4x slower, measured)"""
    return (n + align - 1) // align * align


class BucketedAllReduce:
    def __init__(self, params, bucket_mb=25.0, group=None, reduce_dtype=torch.float32, direct=True):
        self.group = group
        self.direct = direct and reduce_dtype == torch.float32
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        # collectives at world > 1 (QD_DIST_FORCE=1: also on a single-rank group, dev)
        self.collective = self.world > 1 or (_os.environ.get("QD_DIST_FORCE") == "1" and dist.is_initialized())
        params = [p for p in params if p.requires_grad]
        order = list(reversed(params))
        cap = int(bucket_mb * (1 << 20) / 4)
        self.buckets = []  # (flat tensor, [params])
        cur, cur_n = [], 0
        for p in order:
            if cur and cur_n + p.numel() > cap:
                self._make_bucket(cur, cur_n, reduce_dtype)
                cur, cur_n = [], 0
            cur.append(p)
            cur_n += _padded(p.numel())
        if cur:
            self._make_bucket(cur, cur_n, reduce_dtype)
        self.pending = [0] * len(self.buckets)
        self.handles = [None] * len(self.buckets)
        self.hooks = []
        self.bucket_of = {}
        self.view_ptr = {}
        self.taken = set()
        self.sunk = set()
        self._log = []
        for bi, (_, ps) in enumerate(self.buckets):
            for p in ps:
                self.hooks.append(p.register_post_accumulate_grad_hook(self._hook(bi)))
                self.bucket_of[id(p)] = bi
                self.view_ptr[id(p)] = p.grad.data_ptr()
                if self.direct:
                    p._qd_red = self
        self.reset()

    def _make_bucket(self, ps, n, dtype):
        flat = torch.zeros(n, dtype=dtype, device=ps[0].device)
        off = 0
        for p in ps:
            p.grad = flat[off:off + p.numel()].view_as(p)
            off += _padded(p.numel())  # every view 128-B aligned (the library's vectorised folds)
        self.buckets.append((flat, ps))

    def _ready(self, bi):
        self.pending[bi] -= 1
        if self.pending[bi] == 0 and self.collective:
            op = dist.ReduceOp.AVG if dist.get_backend(self.group) == "nccl" else dist.ReduceOp.SUM
            self.handles[bi] = dist.all_reduce(self.buckets[bi][0], op=op, group=self.group, async_op=True)

    def _hook(self, bi):
        def fire(p):
            # the hook also runs for a parameter whose function returned None (a
            # direct write already reported it through ready())
            if id(p) in self.sunk:
                return
            if _DEBUG:
                self._log.append(("hook", id(p), bi, self.pending[bi]))
            self._ready(bi)
        return fire

    def take(self, p):
        """p's bucket view for a direct write, once per step (None if p.grad is no
        longer the bucket view, or p already received a gradient this step)"""
        k = id(p)
        if not self.direct or k in self.taken or p.grad is None or p.grad.data_ptr() != self.view_ptr.get(k):
            return None
        self.taken.add(k)
        return p.grad

    def ready(self, p):
        self.sunk.add(id(p))
        if _DEBUG:
            self._log.append(("sink", id(p), self.bucket_of[id(p)], self.pending[self.bucket_of[id(p)]]))
        self._ready(self.bucket_of[id(p)])

    def reset(self):
        """zero the buckets (the grads) and re-arm the per-bucket counters"""
        for bi, (flat, ps) in enumerate(self.buckets):
            flat.zero_()
            self.pending[bi] = len(ps)
            self.handles[bi] = None
        self.taken.clear()
        self.sunk.clear()

    def finish(self):
        """wait for every bucket's all-reduce; gradients are then the rank mean"""
        for bi, h in enumerate(self.handles):
            if self.collective:
                if h is None:  # a bucket whose params got no gradient this step
                    op = dist.ReduceOp.AVG if dist.get_backend(self.group) == "nccl" else dist.ReduceOp.SUM
                    h = dist.all_reduce(self.buckets[bi][0], op=op, group=self.group, async_op=True)
                h.wait()
                if dist.get_backend(self.group) != "nccl":
                    self.buckets[bi][0].div_(self.world)

    def remove(self):
        for h in self.hooks:
            h.remove()
        for flat, ps in self.buckets:
            for p in ps:
                if getattr(p, "_qd_red", None) is self:
                    del p._qd_red


def broadcast_module(module, src=0, group=None):
    """Copy rank ``src``'s parameters and buffers to every rank (replica start state)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return
    with torch.no_grad():
        for t in list(module.parameters()) + list(module.buffers()):
            dist.broadcast(t.data, src=src, group=group)


def sgd(params, lr=0.1, momentum=0.9, weight_decay=5e-4):
    """The reference sgd_step (trainer.py:50-61) as torch's fused/foreach SGD."""
    return torch.optim.SGD(params, lr=lr, momentum=momentum, weight_decay=weight_decay, dampening=0.0,
                           foreach=True)
