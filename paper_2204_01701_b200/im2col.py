"""Small-channel convs as one fc GEMM over the im2col'd input.

A conv with 3 input channels (the QuadraResNet 7x7/2 stem, the QuadraVGG first
layer) cannot feed the 64-channel-block tcgen05 conv kernels, and zero-padding
the channels to 64 multiplies its work by 21. ``Im2colConv2d`` instead writes
the patches once (``qd_im2col``: col[m][k], k = ky runp + kx C + c with the
filter-row run r*C padded to 8, then zeros to a multiple of 64) and runs the
layer as the same family's *fc* layer over them (ResNet 7x7: runs 21 -> 24,
K 168 -> 192; VGG 3x3: 9 -> 16, 48 -> 64). The weights keep the
reference conv layout (F, C, r, r) and role names; their fc view is a
differentiable permute + pad, so gradients land in the conv-shaped parameters.
The input gradient (col2im) is not implemented: the layer is for data inputs.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F
from torch import nn

from . import _lib
from .errors import DeviceError
from .nn import QuadFunction, _reset
from .spec import QuadraticLayerSpec, param_shapes


def im2col(x, r, s, p, kp):
    """col (N*OH*OW, kp) of an NHWC (channels_last) tensor."""
    n, c, h, w = x.shape
    oh, ow = (h + 2 * p - r) // s + 1, (w + 2 * p - r) // s + 1
    if not x.is_contiguous(memory_format=torch.channels_last):
        x = x.contiguous(memory_format=torch.channels_last)
    col = torch.empty((n * oh * ow, kp), dtype=x.dtype, device=x.device)
    lib = _lib.load()
    st = lib.qd_im2col(n, c, h, w, r, s, p, kp, _lib.BF16 if x.dtype == torch.bfloat16 else _lib.F32,
                       x.data_ptr(), col.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _lib.raise_for(st, "qd_im2col")
    return col, oh, ow


class Im2colConv2d(nn.Module):
    def __init__(self, in_channels, out_channels, kernel_size, stride=1, padding=0, family="proposed", bias=True,
                 device=None, dtype=None):
        super().__init__()
        self.conv_spec = QuadraticLayerSpec(kind="conv", family=family, in_dim=in_channels, out_dim=out_channels,
                                            kernel=kernel_size, stride=stride, pad=padding)
        self.run = kernel_size * in_channels           # the (kx, c) columns of one filter row
        self.runp = (self.run + 7) // 8 * 8             # padded to 16-byte runs (qd_im2col layout)
        self.k = kernel_size * self.runp
        self.kp = (self.k + 63) // 64 * 64
        self.fc_spec = QuadraticLayerSpec(kind="fc", family=family, in_dim=self.kp, out_dim=out_channels)
        fk = dict(device=device, dtype=dtype or torch.float32)
        for role, shape in param_shapes(self.conv_spec).items():
            if role.startswith("b") and not bias:
                self.register_buffer(role, torch.zeros(shape, **fk))
            else:
                setattr(self, role, nn.Parameter(torch.empty(shape, **fk)))
        if device is None or torch.device(device).type != "meta":
            _reset(self, self.conv_spec)

    def fc_tensors(self):
        """The layer's tensors in fc role order: weights as (kp, F), biases as is."""
        out = []
        for role in param_shapes(self.fc_spec):
            t = getattr(self, role)
            if t.dim() == 4:  # (F, C, r, r) -> (r, r C, F) -> zero rows to (r, runp, F) -> (k, F) -> kp
                r = t.shape[2]
                t = t.permute(2, 3, 1, 0).reshape(r, self.run, t.shape[0])
                t = F.pad(t, (0, 0, 0, self.runp - self.run)).reshape(self.k, t.shape[2])
                t = F.pad(t, (0, 0, 0, self.kp - self.k))
            out.append(t)
        return out

    def forward(self, x):
        sp = self.conv_spec
        n, _, h, w = x.shape
        if x.device.type == "meta":
            oh, ow = (h + 2 * sp.pad - sp.kernel) // sp.stride + 1, (w + 2 * sp.pad - sp.kernel) // sp.stride + 1
            return torch.empty((n, sp.out_dim, oh, ow), device=x.device)
        if x.device.type != "cuda":
            raise DeviceError("Im2colConv2d runs on the CUDA kernels only")
        if x.requires_grad:
            raise NotImplementedError("Im2colConv2d: no input gradient (col2im); use it on data inputs")
        col, oh, ow = im2col(x, sp.kernel, sp.stride, sp.pad, self.kp)
        y = QuadFunction.apply(self.fc_spec, None, col, *self.fc_tensors())
        return y.view(n, oh, ow, sp.out_dim).permute(0, 3, 1, 2)  # channels_last NCHW view
