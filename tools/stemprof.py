"""Time the QuadraVGG / ResNet stems (fwd + bwd of weights) in a CUDA graph:
im2col + fc GEMM vs alternatives. python tools/stemprof.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as Fnn
from paper_2204_01701_b200.im2col import Im2colConv2d
from paper_2204_01701_b200.nn import QuadConv2d


class Padded(torch.nn.Module):
    def __init__(self, cin, cout):
        super().__init__()
        self.cin = cin
        self.conv = QuadConv2d(64, cout, 3, 1, 1, "proposed", device="cuda")

    def forward(self, x):
        x = Fnn.pad(x, (0, 0, 0, 0, 0, 64 - self.cin)).contiguous(memory_format=torch.channels_last)
        return self.conv(x)


def timeit(mod, x, reps=20):
    def step():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            y = mod(x)
        y.backward(torch.ones_like(y))
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000


x = torch.randn(256, 3, 32, 32, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
print("vgg stem im2col+fc : %.1f us" % timeit(Im2colConv2d(3, 64, 3, 1, 1, "proposed").cuda(), x))
print("vgg stem padded    : %.1f us" % timeit(Padded(3, 64).cuda(), x))
xr = torch.randn(128, 3, 224, 224, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
print("resnet stem im2col : %.1f us" % timeit(Im2colConv2d(3, 64, 7, 2, 3, "first_order", bias=False).cuda(), xr))
print("resnet stem cudnn  : %.1f us" % timeit(torch.nn.Conv2d(3, 64, 7, 2, 3, bias=False).cuda().to(memory_format=torch.channels_last), xr))

if len(sys.argv) > 1:
    from torch.profiler import ProfilerActivity, profile
    for name, mod, inp in (("vgg", Im2colConv2d(3, 64, 3, 1, 1, "proposed").cuda(), x),
                           ("resnet", Im2colConv2d(3, 64, 7, 2, 3, "first_order", bias=False).cuda(), xr)):
        for _ in range(2):
            with torch.autocast("cuda", dtype=torch.bfloat16):
                y = mod(inp)
            y.backward(torch.ones_like(y))
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            with torch.autocast("cuda", dtype=torch.bfloat16):
                y = mod(inp)
            y.backward(torch.ones_like(y))
            torch.cuda.synchronize()
        print(name)
        for ev in prof.events():
            if ev.device_type == torch.autograd.DeviceType.CUDA:
                print(f"   {ev.device_time_total:8.1f} us  {ev.name[:90]}")
