"""Per-kernel CUDA time of one QuadraNet training step (torch.profiler / CUPTI):
python tools/netprof.py [qvgg16|qresnet18] [batch] [top]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import bench
from paper_2204_01701_b200 import qnets
from paper_2204_01701_b200.optim import QuadSGD

name = sys.argv[1] if len(sys.argv) > 1 else "qvgg16"
builder, batch, hw, classes = bench.NETS[name]
batch = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else batch
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
dev = torch.device("cuda")
torch.backends.cudnn.benchmark = os.environ.get("QD_CUDNN_BENCH", "1") == "1"
torch.manual_seed(0)
model = getattr(qnets, builder)(num_classes=classes).to(dev).to(memory_format=torch.channels_last)
opt = QuadSGD(model, lr=0.01)
x = torch.randn(batch, 3, hw, hw, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
y = torch.randint(0, classes, (batch,), device=dev)


def step():
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = torch.nn.functional.cross_entropy(model(x), y)
    loss.backward()
    opt.step()
    opt.zero_grad(set_to_none=True)


for _ in range(5):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
rows = {}
for ev in prof.events():
    if ev.device_type != torch.autograd.DeviceType.CUDA:
        continue
    k = ev.name[:90]
    t, n = rows.get(k, (0.0, 0))
    rows[k] = (t + ev.device_time_total / 3.0, n + 1)
tot = sum(t for t, _ in rows.values())
print(f"{name} batch {batch}: kernel time per step {tot / 1e3:.3f} ms")
for k, (t, n) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{t / 1e3:8.3f} ms {100 * t / tot:5.1f}%  x{n // 3:<4d} {k}")
