"""Max pooling on the library kernels (qd_maxpool_forward / _backward).

torch.nn.MaxPool2d semantics (floor mode, -inf padding, first maximum wins, NaN
propagates) on NHWC tensors with C % 8 == 0; the backward gathers through a
one-byte window index per output element, so it is deterministic (torch's
scatters with atomics). CUDA channels_last inputs use the kernels; other
devices (CPU inspection, meta-device FLOP counting) use torch's op.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F
from torch import nn

from . import _lib


def _pool_args(x, k, s, p):
    n, c, h, w = x.shape
    return n, c, h, w, k, s, p, (_lib.BF16 if x.dtype == torch.bfloat16 else _lib.F32)


class _MaxPoolFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, k, s, p):
        lib = _lib.load()
        n, c, h, w, k, s, p, dt = _pool_args(x, k, s, p)
        oh, ow = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        y = torch.empty((n, c, oh, ow), dtype=x.dtype, device=x.device, memory_format=torch.channels_last)
        arg = torch.empty((n, oh, ow, c), dtype=torch.uint8, device=x.device)
        st = lib.qd_maxpool_forward(n, c, h, w, k, s, p, dt, x.data_ptr(), y.data_ptr(), arg.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream)
        _lib.raise_for(st, "qd_maxpool_forward")
        ctx.geo = (n, c, h, w, k, s, p, dt)
        ctx.save_for_backward(arg)
        return y

    @staticmethod
    def backward(ctx, dy):
        (arg,) = ctx.saved_tensors
        n, c, h, w, k, s, p, dt = ctx.geo
        lib = _lib.load()
        dy = dy.contiguous(memory_format=torch.channels_last)
        dx = torch.empty((n, c, h, w), dtype=dy.dtype, device=dy.device, memory_format=torch.channels_last)
        st = lib.qd_maxpool_backward(n, c, h, w, k, s, p, dt, dy.data_ptr(), arg.data_ptr(), dx.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream)
        _lib.raise_for(st, "qd_maxpool_backward")
        return dx, None, None, None


class MaxPool2d(nn.MaxPool2d):
    """nn.MaxPool2d (square window, floor mode, no dilation) on the library kernels."""

    def __init__(self, kernel_size, stride=None, padding=0):
        super().__init__(kernel_size, stride, padding)

    def forward(self, x):
        k = self.kernel_size if isinstance(self.kernel_size, int) else self.kernel_size[0]
        s = self.stride if isinstance(self.stride, int) else self.stride[0]
        p = self.padding if isinstance(self.padding, int) else self.padding[0]
        if (x.device.type == "cuda" and x.dim() == 4 and x.shape[1] % 8 == 0
                and x.dtype in (torch.bfloat16, torch.float32)
                and x.is_contiguous(memory_format=torch.channels_last)):
            return _MaxPoolFunction.apply(x, k, s, p)
        return F.max_pool2d(x, k, s, p)
