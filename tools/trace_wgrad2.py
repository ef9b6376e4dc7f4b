"""wgrad2 timeline (CTA 0): QD_TRACE=1 python tools/trace_wgrad2.py"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["QD_TRACE"] = "1"
import torch
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import _lib, neurons
from paper_2204_01701_b200.spec import QuadraticLayerSpec
spec = QuadraticLayerSpec(kind="conv", family="proposed", in_dim=64, out_dim=64, kernel=3, stride=1, pad=1)
x, P, g = Q.synthetic_layer("proposed", "conv", 128, 64, 64, 32, 32, 3, 1, 1, seed=0)
xt = torch.as_tensor(x, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
gt = torch.as_tensor(g, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
params = {k: torch.as_tensor(v, dtype=torch.float32, device="cuda") for k, v in P.items()}
lib = _lib.load()
lib.qd_debug_trace_copy.argtypes = [ctypes.c_void_p]
for _ in range(3):
    y, cache = neurons.forward(spec, params, xt)
    neurons.symbolic_backward(spec, params, cache, gt, want_dx=False)
torch.cuda.synchronize()
buf = np.zeros(8192, dtype=np.uint64)
lib.qd_debug_trace_copy(buf.ctypes.data)
T = buf[:3072].reshape(3, 64, 16).astype(np.int64)
C = buf[3072:4096].reshape(-1, 2).astype(np.int64)
t0 = T[T > 0].min()
for i in range(20):
    p = T[0, i]; m = T[1, i]
    if not (p > 0).any():
        break
    print(f"qb {i:2d}: prod wait {p[0]-t0:7d}->{p[1]-t0:7d} | mma wait {m[0]-t0:7d}->{m[1]-t0:7d} issued {m[2]-t0:7d}")

C = C[C[:, 0] > 0]
t0 = C[:, 0].min()
dur = (C[:, 1] - C[:, 0]) / 1e3
print(f"CTAs {len(C)}: start spread {(C[:,0].max()-t0)/1e3:.2f} us, dur min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us, kernel span {(C[:,1].max()-t0)/1e3:.1f} us")
print("per-CTA durations (us):", " ".join(f"{d:.0f}" for d in dur))
