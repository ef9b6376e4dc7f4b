"""A whole training step as one CUDA graph.

The eager QuadraNet step is host-bound: hundreds of kernel launches issued from
Python (autograd, ctypes calls into the library, the optimizer). ``GraphedStep``
runs the step a few times on a side stream (allocator and library state reach
their steady state: packed weights registered, momentum buffers allocated,
kernel attributes set), captures one more call with ``torch.cuda.graph`` and
afterwards only replays it. Everything the step touches must be static:
parameters, gradient buckets and optimizer state live in fixed buffers (see
``dp.BucketedAllReduce``, ``optim.QuadSGD``), and the inputs are copied into
the graph's own input buffers (``set_inputs``) before a replay.
"""

from __future__ import annotations

import torch


class GraphedStep:
    def __init__(self, step_fn, x, y, warmup=3, counter=None):
        self.x = x.clone()
        self.y = y.clone()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                step_fn(self.x, self.y)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        c0 = counter() if counter else 0
        with torch.cuda.graph(self.graph):
            self.loss = step_fn(self.x, self.y)
        # kernels in one replay, as counted by `counter` (e.g. the library's launch counter)
        self.captured_launches = counter() - c0 if counter else None

    def set_inputs(self, x, y):
        """Stream-ordered copy into the captured input buffers (host or device sources)."""
        self.x.copy_(x, non_blocking=True)
        self.y.copy_(y, non_blocking=True)

    def __call__(self, x=None, y=None):
        if x is not None:
            self.set_inputs(x, y)
        self.graph.replay()
        return self.loss
