"""Per-kernel incremental time (library profile marks, CUDA graph) of one fused
QuadConvBN layer step (forward + backward) at the QuadraResNet-18 shapes:
python tools/qbn_prof.py [N C HW relu res]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01701_b200 import _lib
from paper_2204_01701_b200.bn import QuadConvBN
from paper_2204_01701_b200.nn import QuadConv2d

n, c, hw = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (128, 64, 56)))
res = len(sys.argv) > 5 and sys.argv[5] == "1"
torch.manual_seed(0)
m = QuadConvBN(QuadConv2d(c, c, 3, 1, 1, device="cuda"), relu=not res)
x = torch.randn(n, c, hw, hw, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last).requires_grad_(True)
r = torch.randn(n, c, hw, hw, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
gz = torch.randn(n, c, hw, hw, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)


def step():
    z = m(x, r) if res else m(x)
    z.backward(gz)


for _ in range(3):
    step()
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
lib = _lib.load()
os.environ["QD_NO_PART"] = "1"
os.environ["QD_FOLD_MAIN"] = "1"
g = torch.cuda.CUDAGraph()
lib.qd_profile(1)
with torch.cuda.graph(g):
    lib.qd_profile_mark(torch.cuda.current_stream().cuda_stream)
    step()
lib.qd_profile(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
acc = {}
for rep in range(10):
    flush.fill_(rep)
    g.replay()
    torch.cuda.synchronize()
    seen = {}
    for nm, t in _lib.profile_read():
        k = nm + (f"#{seen.get(nm, 0)}" if seen.get(nm, 0) else "")
        seen[nm] = seen.get(nm, 0) + 1
        acc.setdefault(k, []).append(t)
y_bytes = n * c * hw * hw * 2
print(f"QuadConvBN {n}x{c}x{hw}x{hw} relu={not res} res={res}; |y| = {y_bytes / 1e6:.1f} MB")
tot = 0.0
for k, v in acc.items():
    ms = sorted(v)[len(v) // 2]
    tot += ms
    print(f"  {k:20s} {ms * 1000:8.1f} us  ({y_bytes / (ms * 1e-3) / 1e9:7.0f} GB/s per |y|)")
print(f"  total {tot * 1000:.1f} us")
