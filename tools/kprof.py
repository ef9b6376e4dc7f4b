"""Per-kernel times of one layer step via the library's event marks.
python tools/kprof.py [workload=c2] [flush=1] [reps=10]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import _lib, neurons
wl_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
flush_on = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
wl = bench.WORKLOADS[wl_name]
fam, kind, n, c, f, h, w, r, s, p, dts = wl
spec = bench.make_spec(wl)
x64, P64, g64 = Q.synthetic_layer(fam, kind, n, c, f, h, w, r, s, p, seed=0)
dev = "cuda"
x = torch.as_tensor(x64, device=dev).bfloat16().contiguous(memory_format=torch.channels_last)
gy = torch.as_tensor(g64, device=dev).bfloat16().contiguous(memory_format=torch.channels_last)
params = {k: torch.as_tensor(v, dtype=torch.float32, device=dev) for k, v in P64.items()}
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
lib = _lib.load()
want_dx = not (len(sys.argv) > 4 and sys.argv[4] == "nodx")
def step():
    y, cache = neurons.forward(spec, params, x)
    neurons.symbolic_backward(spec, params, cache, gy, want_dx=want_dx)
for _ in range(3):
    step()
torch.cuda.synchronize()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    step()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
lib.qd_profile(1)
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    lib.qd_profile_mark(torch.cuda.current_stream().cuda_stream)
    step()
lib.qd_profile(0)
acc = {}
for i in range(reps):
    if flush_on:
        bench.flush_l2(flush, i)
    graph.replay()
    torch.cuda.synchronize()
    seen = {}
    for nm, t in _lib.profile_read():
        k = nm
        if nm in ("conv2", "conv_gemm"):
            k = nm + ("[fprop]" if seen.get(nm, 0) == 0 else "[dgrad]")
            seen[nm] = seen.get(nm, 0) + 1
        acc.setdefault(k, []).append(t)
print(wl_name, "flush" if flush_on else "warm", " ".join(f"{k}={1000*sum(v)/len(v):.1f}us" for k, v in acc.items()))
