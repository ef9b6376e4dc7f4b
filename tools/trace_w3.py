"""wgrad3 stage timeline of CTA 0 (QD_TRACE): producer empty-wait start/end, MMA
full-wait start/end and issue end per q block, in SM cycles. QD_NO_PART=1 for
the kernel alone on all SMs. python tools/trace_w3.py [workload]"""
import ctypes, os, sys
os.environ["QD_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import _lib, neurons
lib = _lib.load()
lib.qd_debug_trace_copy.argtypes = [ctypes.c_void_p]
wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
fam, kind, n, c, f, h, w, r, s, p, dts = wl
spec = bench.make_spec(wl)
x64, P64, g64 = Q.synthetic_layer(fam, kind, n, c, f, h, w, r, s, p, seed=0)
x = torch.as_tensor(x64, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
gy = torch.as_tensor(g64, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
params = {k: torch.as_tensor(v, dtype=torch.float32, device="cuda") for k, v in P64.items()}
for _ in range(5):
    y, cache = neurons.forward(spec, params, x)
    neurons.symbolic_backward(spec, params, cache, gy, want_dx=False)
torch.cuda.synchronize()
buf = np.zeros(8192, dtype=np.uint64)
lib.qd_debug_trace_copy(buf.ctypes.data)
T = buf[:2048].reshape(2, 64, 16).astype(np.int64)
t0 = T[T > 0].min()
prev = None
for blk in range(64):
    pe, me = T[0, blk], T[1, blk]
    if me[1] == 0:
        break
    row = (f"blk {blk:2d}: prod wait {pe[0]-t0:7d}->{pe[1]-t0:7d} | mma wait {me[0]-t0:7d}->{me[1]-t0:7d} "
           f"(stall {me[1]-me[0]:5d}) issue end {me[2]-t0:7d} (issue {me[2]-me[1]:5d})")
    if prev is not None:
        row += f" block {me[1]-prev:5d}"
    prev = me[1]
    print(row)
