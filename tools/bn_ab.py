"""A/B of the BN kernels (QD_BN_OLD=1: register-streaming kernels + finalize
launches; default: bulk-copy streaming with in-kernel grid folds) on the
QuadraResNet-18 BN shapes: forward (stats + apply) and forward + backward of
BNAct2d, CUDA-graph replays, L2 flushed before each replay."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01701_b200.bn import BNAct2d, bn_forward

shapes = [(128, 64, 112), (128, 64, 56), (128, 128, 28), (128, 256, 14), (128, 512, 7)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1000)
    return sorted(ts)[len(ts) // 2]


for n, c, hw in shapes:
    x = torch.randn(n, c, hw, hw, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    gz = torch.randn_like(x)
    m = BNAct2d(c, relu=True).cuda()
    out = []
    for mode in ("old", "new"):
        if mode == "old":
            os.environ["QD_BN_OLD"] = "1"
        else:
            os.environ.pop("QD_BN_OLD", None)
        fwd = lambda: bn_forward(x, m.weight, m.bias, m.running_mean, m.running_var, 0.1, 1e-5, True, True)  # noqa
        x1 = x.detach().clone().requires_grad_(True)

        def step():
            z = m(x1)
            z.backward(gz)
        out.append((timed(fwd), timed(step)))
    yb = x.numel() * 2
    print(f"{n}x{c}x{hw}x{hw} |y|={yb/1e6:.1f} MB  fwd old {out[0][0]:6.1f} new {out[1][0]:6.1f} us "
          f"({3 * yb / out[1][0] / 1e3:5.0f} GB/s) | fwd+bwd old {out[0][1]:6.1f} new {out[1][1]:6.1f} us "
          f"({8 * yb / out[1][1] / 1e3:5.0f} GB/s)")
