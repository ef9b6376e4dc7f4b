"""Timeline of conv2 (cluster 0, CTA 0): QD_TRACE=1 python tools/trace_conv2.py [fprop|dgrad]"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["QD_TRACE"] = "1"
import torch
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import _lib, neurons
from paper_2204_01701_b200.spec import QuadraticLayerSpec
which = sys.argv[1] if len(sys.argv) > 1 else "fprop"
fam = sys.argv[2] if len(sys.argv) > 2 else "proposed"
n_, c_, hw_ = (int(v) for v in (sys.argv[3:6] if len(sys.argv) > 5 else (128, 64, 32)))
spec = QuadraticLayerSpec(kind="conv", family=fam, in_dim=c_, out_dim=c_, kernel=3, stride=1, pad=1)
x, P, g = Q.synthetic_layer(fam, "conv", n_, c_, c_, hw_, hw_, 3, 1, 1, seed=0)
xt = torch.as_tensor(x, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
gt = torch.as_tensor(g, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
params = {k: torch.as_tensor(v, dtype=torch.float32, device="cuda") for k, v in P.items()}
lib = _lib.load()
lib.qd_debug_trace_copy.argtypes = [ctypes.c_void_p]
for _ in range(3):
    y, cache = neurons.forward(spec, params, xt)
    if which == "dgrad":
        neurons.symbolic_backward(spec, params, cache, gt, want_dw=False)
torch.cuda.synchronize()
buf = np.zeros(8192, dtype=np.uint64)
lib.qd_debug_trace_copy(buf.ctypes.data)
T = buf[:4096].reshape(4, 64, 16).astype(np.int64)
t0 = T[T > 0].min()
names = {0: "producer", 1: "mma", 2: "epilogue", 3: "xform"}
for tile in range(10):
    row = []
    for role in range(4):
        ev = T[role, tile]
        nz = [(i, int(v - t0)) for i, v in enumerate(ev) if v > 0]
        row.append(f"{names[role]}: " + " ".join(f"{i}@{v}" for i, v in nz))
    print(f"tile {tile}: " + " | ".join(row))
G = buf[4096:6144].reshape(-1, 2).astype(np.int64)
K = buf[6144:8192].reshape(-1, 2).astype(np.int64)
nb = int((G[:, 0] > 0).sum())
G, K = G[:nb], K[:nb]
dur = (G[:, 1] - G[:, 0]) / 1e3
ghz = (K[:, 1] - K[:, 0]) / (G[:, 1] - G[:, 0])
print(f"CTAs {nb}: start spread {(G[:,0].max()-G[:,0].min())/1e3:.2f} us, span {(G[:,1].max()-G[:,0].min())/1e3:.1f} us, "
      f"dur min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us, clock med {np.median(ghz):.3f} GHz")
