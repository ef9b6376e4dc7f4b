"""One C2 layer step (pack + fwd + bwd) for profiling: python tools/prof_step.py [iters] [family] [bf16|fp32]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import neurons
from paper_2204_01701_b200.spec import QuadraticLayerSpec
it = int(sys.argv[1]) if len(sys.argv) > 1 else 3
fam = sys.argv[2] if len(sys.argv) > 2 else "proposed"
n, c, f, h = 128, 64, 64, 32
dt = torch.float32 if len(sys.argv) > 3 and sys.argv[3] == "fp32" else torch.bfloat16
spec = QuadraticLayerSpec(kind="conv", family=fam, in_dim=c, out_dim=f, kernel=3, stride=1, pad=1)
x, P, g = Q.synthetic_layer(fam, "conv", n, c, f, h, h, 3, 1, 1, seed=0)
dev = "cuda"
xt = torch.as_tensor(x, device=dev).to(dt).contiguous(memory_format=torch.channels_last)
gt = torch.as_tensor(g, device=dev).to(dt).contiguous(memory_format=torch.channels_last)
params = {k: torch.as_tensor(v, dtype=torch.float32, device=dev) for k, v in P.items()}
for _ in range(it):
    y, cache = neurons.forward(spec, params, xt, dtype=dt)
    grads, dx = neurons.symbolic_backward(spec, params, cache, gt)
torch.cuda.synchronize()
print("ok")
