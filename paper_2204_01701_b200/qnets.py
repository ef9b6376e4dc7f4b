"""QuadraResNet-18 and QuadraVGG-16 (BASELINE.json configs 3 and 4).

The reference cannot express these nets (its ModelConfig is a plain chain
with no pooling or residual ops, /root/reference/pkg/src/quadra/autobuild.py:75-118,
model.py:151-155), so they are built here in torch around
the quadratic conv module; every 3x3 conv is a ``QuadConv2d`` (proposed
neuron by default). Around them: BN (+ReLU) and max-pool on the library's
kernels (``bn.BNAct2d``, ``pool.MaxPool2d``), the 3-channel stems as one fc
GEMM over im2col'd patches (``im2col.Im2colConv2d``), the 1x1 shortcuts,
residual adds, pooling head and loss in torch:

* QuadraVGG-16 (CIFAR, 3x32x32, 10 classes): VGG-16 "D" layout, all 13 convs
  quadratic, each followed by BatchNorm + ReLU, five 2x2 max-pools, a
  512 -> 10 linear head. 44.16 M parameters (matches the
  paper's 4.41E+7).
* QuadraResNet-18 (ImageNet, 3x224x224, 1000 classes): first-order 7x7/2
  stem + BN + ReLU + 3x3/2 max-pool, BasicBlocks [2, 2, 2, 2] at widths
  64/128/256/512 whose 3x3 convs are quadratic (3 of them stride 2), 1x1/2
  first-order downsample + BN, global average pool, 512 -> 1000 linear.

Activations are bf16 channels_last; parameters are fp32 masters. Run the
forward under ``torch.autocast("cuda", torch.bfloat16)`` so the first-order
layers compute in bf16 too (batch norm keeps fp32 statistics).
"""

from __future__ import annotations

import torch
from torch import nn

from .bn import BNAct2d, QuadConvBN
from .nn import QuadConv2d
from .im2col import Im2colConv2d
from .pool import MaxPool2d


def quad_conv(cin, cout, k=3, s=1, p=1, family="proposed"):
    if cin % 64:  # few input channels (a stem): one fc GEMM over the im2col'd input
        return Im2colConv2d(cin, cout, k, s, p, family)
    return QuadConv2d(cin, cout, k, s, p, family)


VGG16_CFG = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]


class QuadraVGG16(nn.Module):
    def __init__(self, num_classes=10, family="proposed"):
        super().__init__()
        layers = []
        cin = 3
        for v in VGG16_CFG:
            if v == "M":
                layers.append(MaxPool2d(2, 2))
            elif cin % 64:  # 3-channel stem (im2col + fc GEMM), then BN + ReLU (one node; Identity keeps indices)
                layers += [quad_conv(cin, v, 3, 1, 1, family), BNAct2d(v, relu=True), nn.Identity()]
                cin = v
            else:  # quad conv -> BN -> ReLU as one fused node (bn.QuadConvBN)
                layers.append(QuadConvBN(QuadConv2d(cin, v, 3, 1, 1, family), relu=True))
                cin = v
        self.features = nn.Sequential(*layers)
        self.classifier = nn.Linear(512, num_classes)

    def forward(self, x):
        x = self.features(x)
        return self.classifier(torch.flatten(x, 1))


class QuadBasicBlock(nn.Module):
    expansion = 1

    def __init__(self, inplanes, planes, stride=1, family="proposed"):
        super().__init__()
        # conv -> BN (-> ReLU) fused (bn.QuadConvBN; stride 2 runs its unfused form)
        self.cbr1 = QuadConvBN(quad_conv(inplanes, planes, 3, stride, 1, family), relu=True)
        self.cb2 = QuadConvBN(quad_conv(planes, planes, 3, 1, 1, family), relu=False)
        self.relu = nn.ReLU(inplace=True)
        self.down = None
        if stride != 1 or inplanes != planes:
            # 1x1 (stride 2) shortcut + BN as one node on the library kernels (first-order
            # family; its bias cancels in the BN like the quadratic layers' biases)
            self.down = QuadConvBN(quad_conv(inplanes, planes, 1, stride, 0, "first_order"), relu=False)

    def forward(self, x):
        idt = x if self.down is None else self.down(x)
        # cb2's BN apply also adds the identity and applies the block's ReLU
        return self.cb2(self.cbr1(x), idt)


class QuadraResNet18(nn.Module):
    def __init__(self, num_classes=1000, family="proposed"):
        super().__init__()
        # first-order stem; BN + ReLU as one node on the library kernels (Identity keeps indices)
        self.stem = nn.Sequential(Im2colConv2d(3, 64, 7, 2, 3, family="first_order", bias=False),
                                  BNAct2d(64, relu=True), nn.Identity(), MaxPool2d(3, 2, 1))
        blocks = []
        inplanes = 64
        for planes, stride in ((64, 1), (128, 2), (256, 2), (512, 2)):
            for i in range(2):
                blocks.append(QuadBasicBlock(inplanes, planes, stride if i == 0 else 1, family))
                inplanes = planes
        self.layers = nn.Sequential(*blocks)
        self.pool = nn.AdaptiveAvgPool2d(1)
        self.fc = nn.Linear(512, num_classes)

    def forward(self, x):
        x = self.layers(self.stem(x))
        return self.fc(torch.flatten(self.pool(x), 1))


def quad_layers(model):
    return [m for m in model.modules() if isinstance(m, QuadConv2d)]


def count_params(model):
    return sum(p.numel() for p in model.parameters())
