"""fp64 CPU composition of QuadraVGG-16 / QuadraResNet-18 -- TEST INFRASTRUCTURE ONLY.

Secondary oracle of SURVEY.md §8(c) "Gaps": the reference cannot express
these nets (no pooling / residual / average pool; autobuild.py:75-118,
model.py:151-155), so one training step of each is restated here in float64
torch on the CPU, op by op, with autograd for the chain rule:

* quadratic layer (proposed): ``y = (Wa x + ba)(Wb x + bb) + Wc x + bc``
  (reference neurons.py:268-274; conv as a cross-correlation, tensor.py:313-320);
  the per-layer formula is pinned against ``quadra_oracle`` (itself pinned to
  the reference's golden vectors) by tests/test_net_oracle.py;
* first-order conv ``W x + b`` (neurons.py:242-244);
* batch norm, training mode, BIASED batch variance (tensor.py:440-450),
  eps 1e-5 (model.py:23-24); ReLU (tensor.py:251-254);
* max pool / average pool / linear head: the standard definitions;
* cross-entropy, mean over the batch (tensor.py:475-496).

Parameters are read by name from a state dict laid out like the product's
modules (``paper_2204_01701_b200.qnets``); the structure below is written
independently from the net definitions of BASELINE.json configs 3 and 4.
Only tests/ may import this module.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F

VGG16_CFG = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]


def quad_conv(x, P, pre, family, stride, pad):
    """Quadratic (or first-order) conv layer from the parameters under ``pre``."""
    conv = lambda w: F.conv2d(x, w, stride=stride, padding=pad)  # noqa: E731
    if family == "first_order":
        y = conv(P[pre + "W"])
        b = P.get(pre + "b")
        return y if b is None else y + b.view(1, -1, 1, 1)
    if family != "proposed":
        raise ValueError(family)
    a = conv(P[pre + "Wa"]) + P[pre + "ba"].view(1, -1, 1, 1)
    b = conv(P[pre + "Wb"]) + P[pre + "bb"].view(1, -1, 1, 1)
    return a * b + conv(P[pre + "Wc"]) + P[pre + "bc"].view(1, -1, 1, 1)


def batchnorm(y, gamma, beta, eps=1e-5):
    """training-mode BN with the biased batch variance (tensor.py:440-450)."""
    mean = y.mean(dim=(0, 2, 3), keepdim=True)
    var = ((y - mean) ** 2).mean(dim=(0, 2, 3), keepdim=True)
    return (y - mean) / torch.sqrt(var + eps) * gamma.view(1, -1, 1, 1) + beta.view(1, -1, 1, 1)


def vgg16_logits(P, x):
    i = 0
    cin = x.shape[1]
    h = x
    for v in VGG16_CFG:
        if v == "M":
            h = F.max_pool2d(h, 2, 2)
            i += 1
        elif cin % 64:  # stem: quadratic conv (im2col'd in the product), BN + ReLU, Identity
            h = quad_conv(h, P, f"features.{i}.", "proposed", 1, 1)
            h = torch.relu(batchnorm(h, P[f"features.{i + 1}.weight"], P[f"features.{i + 1}.bias"]))
            i += 3
            cin = v
        else:  # quadratic conv -> BN -> ReLU node
            h = quad_conv(h, P, f"features.{i}.layer.", "proposed", 1, 1)
            h = torch.relu(batchnorm(h, P[f"features.{i}.weight"], P[f"features.{i}.bias"]))
            i += 1
            cin = v
    h = torch.flatten(h, 1)
    return h @ P["classifier.weight"].T + P["classifier.bias"]


def resnet18_logits(P, x):
    h = quad_conv(x, P, "stem.0.", "first_order", 2, 3)
    h = torch.relu(batchnorm(h, P["stem.1.weight"], P["stem.1.bias"]))
    h = F.max_pool2d(h, 3, 2, 1)
    inplanes, bi = 64, 0
    for planes, stride in ((64, 1), (128, 2), (256, 2), (512, 2)):
        for k in range(2):
            s = stride if k == 0 else 1
            pre = f"layers.{bi}."
            t = quad_conv(h, P, pre + "cbr1.layer.", "proposed", s, 1)
            t = torch.relu(batchnorm(t, P[pre + "cbr1.weight"], P[pre + "cbr1.bias"]))
            t = quad_conv(t, P, pre + "cb2.layer.", "proposed", 1, 1)
            t = batchnorm(t, P[pre + "cb2.weight"], P[pre + "cb2.bias"])
            if s != 1 or inplanes != planes:
                idt = quad_conv(h, P, pre + "down.layer.", "first_order", s, 0)
                idt = batchnorm(idt, P[pre + "down.weight"], P[pre + "down.bias"])
            else:
                idt = h
            h = torch.relu(t + idt)
            inplanes = planes
            bi += 1
    h = h.mean(dim=(2, 3))
    return h @ P["fc.weight"].T + P["fc.bias"]


def train_step_grads(net, params, x, labels):
    """(logits, loss, {name: grad}) of one training step in fp64.

    ``params``: name -> tensor (any dtype / device; copied to fp64 CPU leaves);
    ``x``: NCHW images; ``labels``: int64 class indices. Mean cross-entropy
    (tensor.py:475-496)."""
    P = {k: v.detach().to("cpu", torch.float64).clone().requires_grad_(True) for k, v in params.items()}
    xx = x.detach().to("cpu", torch.float64)
    fn = {"qvgg16": vgg16_logits, "qresnet18": resnet18_logits}[net]
    logits = fn(P, xx)
    loss = F.cross_entropy(logits, labels.detach().cpu())
    loss.backward()
    return logits.detach(), float(loss), {k: (v.grad if v.grad is not None else torch.zeros_like(v))
                                          for k, v in P.items()}
