"""Stem conv (7x7 s2 p3, 3 -> 64, batch 128, 224^2, bf16 channels_last): our
im2col + GEMM path vs torch/cuDNN conv2d, forward + weight gradient, CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01701_b200.im2col import Im2colConv2d

torch.backends.cudnn.benchmark = True
dev = torch.device("cuda")
x = torch.randn(128, 3, 224, 224, device=dev).bfloat16().contiguous(memory_format=torch.channels_last)
ours = Im2colConv2d(3, 64, 7, 2, 3, family="first_order", bias=False).to(dev)
conv = torch.nn.Conv2d(3, 64, 7, 2, 3, bias=False).to(dev).to(memory_format=torch.channels_last)
g = torch.randn(128, 64, 112, 112, device=dev).bfloat16().contiguous(memory_format=torch.channels_last)


def run_ours():
    y = ours(x)
    y.backward(g)


def run_cudnn():
    with torch.autocast("cuda", dtype=torch.bfloat16):
        y = conv(x)
    y.backward(g)


for name, fn in (("ours", run_ours), ("cudnn", run_cudnn)):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(name, round(a.elapsed_time(b) / 20, 3), "ms per fwd + wgrad")
