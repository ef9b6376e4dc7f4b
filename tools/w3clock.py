"""Per-CTA duration and SM clock of wgrad3 inside repeated steps (QD_TRACE)."""
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
def step():
    y, cache = neurons.forward(spec, params, x)
    neurons.symbolic_backward(spec, params, cache, gy, want_dx=False)
for _ in range(50):
    step()
torch.cuda.synchronize()
buf = np.zeros(8192, dtype=np.uint64)
lib.qd_debug_trace_copy(buf.ctypes.data)
G = buf[3072:4096].reshape(-1, 2).astype(np.int64)
C = buf[2048:3072].reshape(-1, 2).astype(np.int64)
nb = int((G[:, 0] > 0).sum())
G, C = G[:nb], C[:nb]
dur = (G[:, 1] - G[:, 0]) / 1e3
cyc = C[:, 1] - C[:, 0]
print(f"CTAs {nb}: start spread {(G[:,0].max()-G[:,0].min())/1e3:.2f} us, span {(G[:,1].max()-G[:,0].min())/1e3:.1f} us,"
      f" dur min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us")
ghz = cyc / (G[:, 1] - G[:, 0])
print(f"SM clock in-kernel: min/med/max {ghz.min():.3f}/{np.median(ghz):.3f}/{ghz.max():.3f} GHz")

Dn = buf[4096:4096 + nb].astype(np.int64)
if (Dn > 0).all():
    epi = (G[:, 1] - Dn) / 1e3
    main = (Dn - G[:, 0]) / 1e3
    print(f"main loop min/med/max {main.min():.1f}/{np.median(main):.1f}/{main.max():.1f} us, "
          f"epilogue min/med/max {epi.min():.1f}/{np.median(epi):.1f}/{epi.max():.1f} us")
T = buf[:3072].reshape(3, 64, 16).astype(np.int64)
t0 = T[0, 0, 0] if T[0, 0, 0] > 0 else T[T > 0].min()
print("CTA0 per q block (cycles from first event): prod[acq empty] mma[full acquired, issued]")
prev = None
for blk in range(64):
    pe, m1, m2 = T[0, blk, 1], T[1, blk, 1], T[1, blk, 2]
    if m2 == 0:
        break
    d = "" if prev is None else f" period {m1 - prev}"
    print(f"  blk {blk:2d}: prod {pe - t0:6d}  mma full@{m1 - t0:6d} issued@{m2 - t0:6d} (issue {m2 - m1}){d}")
    prev = m1
