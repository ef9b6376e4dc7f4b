"""BN kernels alone: BNAct2d (BN + ReLU, first-order) forward + backward in a CUDA
graph, per shape; reports us and the effective bandwidth of the 5 passes
(fwd: stats read y, apply read y + write z; bwd: reduce read y + dz, emit read
y + dz + write dy). python tools/bnbench.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01701_b200.bn import BNAct2d

SHAPES = [(128, 64, 112), (128, 64, 56), (128, 128, 28), (128, 256, 14), (128, 512, 7)]


def bench(n, c, h, reps=20):
    m = BNAct2d(c, relu=True).cuda()
    x = torch.randn(n, c, h, h, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    x.requires_grad_(True)
    gz = torch.randn(n, c, h, h, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)

    def step():
        z = m(x)
        z.backward(gz)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1000
    nbytes = x.numel() * 2 * (1 + 2 + 2 + 3)  # 8 element-passes
    return us, nbytes / (us * 1e-6) / 1e12


tot = 0.0
for sh in SHAPES:
    us, tbs = bench(*sh)
    tot += us
    print(f"BN+ReLU fwd+bwd {sh}: {us:7.1f} us  {tbs:5.2f} TB/s effective")
print(f"sum {tot:.1f} us")

if len(sys.argv) > 1:
    from torch.profiler import ProfilerActivity, profile
    n, c, h = (int(v) for v in sys.argv[1:4])
    m = BNAct2d(c, relu=True).cuda()
    x = torch.randn(n, c, h, h, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    x.requires_grad_(True)
    gz = torch.randn(n, c, h, h, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    for _ in range(3):
        m(x).backward(gz)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        m(x).backward(gz)
        torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    for e in evs:
        print(f"  {e.time_range.start - t0:8.1f} +{e.time_range.end - e.time_range.start:6.1f} us  {e.name[:80]}")
