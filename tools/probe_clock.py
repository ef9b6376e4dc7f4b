"""SM clock under load: spin kernel (clock64 vs globaltimer vs CUDA events), alone and
right after a C2 step graph. python tools/probe_clock.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import _lib, neurons
lib = _lib.load()
lib.qd_debug_spin.argtypes = [ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p]
out = torch.zeros(4, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
def spin(cyc):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    lib.qd_debug_spin(cyc, out.data_ptr(), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    c0, c1, t0, t1 = [int(v) for v in out.cpu()]
    ev = e0.elapsed_time(e1) * 1e3
    print(f"spin {cyc}: clock {c1-c0} cyc, globaltimer {(t1-t0)/1e3:.1f} us, events {ev:.1f} us -> "
          f"{(c1-c0)/(t1-t0):.3f} GHz (gtimer), {(c1-c0)/ev/1e3:.3f} GHz (events)")
for _ in range(2):
    spin(200000)
wl = bench.WORKLOADS["c2"]
fam, kind, n, c, f, h, w, r, s, p, dts = wl
spec = bench.make_spec(wl)
x64, P64, g64 = Q.synthetic_layer(fam, kind, n, c, f, h, w, r, s, p, seed=0)
x = torch.as_tensor(x64, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
gy = torch.as_tensor(g64, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
params = {k: torch.as_tensor(v, dtype=torch.float32, device="cuda") for k, v in P64.items()}
def step():
    y, cache = neurons.forward(spec, params, x)
    neurons.symbolic_backward(spec, params, cache, gy)
for _ in range(3):
    step()
torch.cuda.synchronize()
for k in (10, 200, 2000):
    for _ in range(k):
        step()
    # spin right behind the queued steps: measures the clock the steps left the GPU at
    spin(200000)
