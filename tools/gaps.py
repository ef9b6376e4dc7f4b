"""Kernel timeline of one CUDA-graph replay of a QuadraNet training step:
largest idle gaps between consecutive kernels. python tools/gaps.py [qvgg16|qresnet18] [top]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import bench
from paper_2204_01701_b200 import qnets
from paper_2204_01701_b200.dp import BucketedAllReduce
from paper_2204_01701_b200.graphstep import GraphedStep
from paper_2204_01701_b200.optim import QuadSGD

name = sys.argv[1] if len(sys.argv) > 1 else "qvgg16"
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
builder, batch, hw, classes = bench.NETS[name]
torch.backends.cudnn.benchmark = True
torch.manual_seed(0)
model = getattr(qnets, builder)(num_classes=classes).cuda().to(memory_format=torch.channels_last)
opt = QuadSGD(model, lr=0.01)
red = BucketedAllReduce(model.parameters())
x = torch.randn(batch, 3, hw, hw, device="cuda").to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
y = torch.randint(0, classes, (batch,), device="cuda")


def step(xb, yb):
    red.reset()
    with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
        loss = torch.nn.functional.cross_entropy(model(xb), yb)
    loss.backward()
    red.finish()
    opt.step()
    return loss


gs = GraphedStep(step, x, y)
for _ in range(3):
    gs()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    gs()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
t0, t1 = evs[0].time_range.start, max(e.time_range.end for e in evs)
busy = 0.0
gaps = []
end = evs[0].time_range.start
for i, e in enumerate(evs):
    if e.time_range.start > end:
        gaps.append((e.time_range.start - end, evs[i - 1].name[:60] if i else "", e.name[:60]))
    end = max(end, e.time_range.end)
print(f"{name}: span {(t1 - t0) / 1e3:.3f} ms, {len(evs)} kernels, idle {sum(g[0] for g in gaps) / 1e3:.3f} ms "
      f"in {len(gaps)} gaps")
for g, a, b in sorted(gaps, reverse=True)[:top]:
    print(f"  {g:8.1f} us  after {a}  before {b}")
# per-kernel totals of the same replay
tot = {}
for e in evs:
    k = e.name[:90]
    t, c = tot.get(k, (0.0, 0))
    tot[k] = (t + (e.time_range.end - e.time_range.start), c + 1)
print(f"kernel time {sum(t for t, _ in tot.values()) / 1e3:.3f} ms (overlapping streams counted twice)")
for k, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:int(os.environ.get("GAPS_TOP", "45"))]:
    print(f"  {t / 1e3:7.3f} ms  x{c:<4d} {k}")
