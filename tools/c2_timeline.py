"""Kernel timeline (start/end, us) of one CUDA-graph replay of a layer step:
python tools/c2_timeline.py [workload=c2] [pdl=1]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import bench
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import neurons

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
fam, kind, n, c, f, h, w, r, s, p, dts = wl
spec = bench.make_spec(wl)
x64, P64, g64 = Q.synthetic_layer(fam, kind, n, c, f, h, w, r, s, p, seed=0)
_dt = torch.bfloat16 if dts == "bf16" else torch.float32
_fmt = torch.channels_last if kind != "fc" else torch.contiguous_format
x = torch.as_tensor(x64, device="cuda").to(_dt).contiguous(memory_format=_fmt)
gy = torch.as_tensor(g64, device="cuda").to(_dt).contiguous(memory_format=_fmt)
params = {k: torch.as_tensor(v, dtype=torch.float32, device="cuda") for k, v in P64.items()}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def step():
    y, cache = neurons.forward(spec, params, x)
    neurons.symbolic_backward(spec, params, cache, gy)


for _ in range(3):
    step()
torch.cuda.synchronize()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    step()
torch.cuda.current_stream().wait_stream(side)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
for rep in range(2):
    bench.flush_l2(flush, rep)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g.replay()
        torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    print(f"--- replay {rep}: span {(max(e.time_range.end for e in evs) - t0):.1f} us")
    for e in evs:
        print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} {e.time_range.end - e.time_range.start:7.1f}  {e.name[:70]}")
