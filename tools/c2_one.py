"""One conv2 fprop (+ optional dgrad) for compute-sanitizer / quick checks:
python tools/c2_one.py [N C F H W] [bwd]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import neurons
from paper_2204_01701_b200.spec import QuadraticLayerSpec
a = [int(v) for v in sys.argv[1:6]] if len(sys.argv) > 5 else [4, 64, 64, 12, 12]
n, c, f, h, w = a
spec = QuadraticLayerSpec(kind="conv", family="proposed", in_dim=c, out_dim=f, kernel=3, stride=1, pad=1)
x, P, g = Q.synthetic_layer("proposed", "conv", n, c, f, h, w, 3, 1, 1, seed=0, random_bias=True)
xt = torch.as_tensor(x, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
gt = torch.as_tensor(g, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
params = {k: torch.as_tensor(v, dtype=torch.float32, device="cuda") for k, v in P.items()}
y, cache = neurons.forward(spec, params, xt)
torch.cuda.synchronize()
print("fprop ok", float(y.float().abs().sum()))
if "bwd" in sys.argv:
    grads, dx = neurons.symbolic_backward(spec, params, cache, gt)
    torch.cuda.synchronize()
    print("bwd ok", float(dx.float().abs().sum()))
