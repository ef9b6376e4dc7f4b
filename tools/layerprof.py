"""All CUDA kernels (ours and torch's) of one layer step of a bench workload:
python tools/layerprof.py <workload> [top]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import bench
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import neurons

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
fam, kind, n, c, f, h, w, r, s, p, dts = wl
spec = bench.make_spec(wl)
x64, P64, g64 = Q.synthetic_layer(fam, kind, n, c, f, h, w, r, s, p, seed=0)
dt = torch.bfloat16 if dts == "bf16" else torch.float32
x = torch.as_tensor(x64, device="cuda").to(dt)
gy = torch.as_tensor(g64, device="cuda").to(dt)
if kind != "fc":
    x = x.contiguous(memory_format=torch.channels_last)
    gy = gy.contiguous(memory_format=torch.channels_last)
params = {k: torch.as_tensor(v, dtype=torch.float32, device="cuda") for k, v in P64.items()}


def step():
    y, cache = neurons.forward(spec, params, x, dtype=dt)
    neurons.symbolic_backward(spec, params, cache, gy)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        step()
    torch.cuda.synchronize()
rows = {}
for ev in prof.events():
    if ev.device_type != torch.autograd.DeviceType.CUDA:
        continue
    k = ev.name[:80]
    t, cnt = rows.get(k, (0.0, 0))
    rows[k] = (t + ev.device_time_total / 5.0, cnt + 1)
tot = sum(t for t, _ in rows.values())
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'c2'}: kernel time per step {tot:.1f} us")
for k, (t, cnt) in sorted(rows.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{t:8.1f} us  x{cnt // 5:<3d} {k}")
