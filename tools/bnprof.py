"""Per-kernel times of one fused QuadConvBN layer step vs the unfused composition."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01701_b200 import _lib
from paper_2204_01701_b200.bn import QuadConvBN
from paper_2204_01701_b200.nn import QuadConv2d
n, c, h = [int(v) for v in sys.argv[1:4]] if len(sys.argv) > 3 else (128, 64, 56)
layer = QuadConv2d(c, c, 3, 1, 1, device="cuda")
mod = QuadConvBN(layer, relu=True)
bn = torch.nn.BatchNorm2d(c).cuda().to(memory_format=torch.channels_last)
x = torch.randn(n, c, h, h, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last).requires_grad_(True)
gz = torch.randn(n, c, h, h, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
lib = _lib.load()
def fused():
    z = mod(x); z.backward(gz)
def unfused():
    with torch.autocast("cuda", dtype=torch.bfloat16):
        z = torch.relu(bn(layer(x)))
    z.backward(gz)
for name, fn in (("fused", fused), ("unfused", unfused)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record(); torch.cuda.synchronize()
    print(name, round(e0.elapsed_time(e1) / 10 * 1000, 1), "us/step")
