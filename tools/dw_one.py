"""One depth-wise layer step for profiling: python tools/dw_one.py [family] [N C H]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import neurons
from paper_2204_01701_b200.spec import QuadraticLayerSpec
fam = sys.argv[1] if len(sys.argv) > 1 else "proposed"
n, c, h = [int(v) for v in sys.argv[2:5]] if len(sys.argv) > 4 else (64, 256, 28)
spec = QuadraticLayerSpec(kind="dwconv", family=fam, in_dim=c, out_dim=c, kernel=3, stride=1, pad=1)
x, P, g = Q.synthetic_layer(fam, "dwconv", n, c, c, h, h, 3, 1, 1, seed=0)
xt = torch.as_tensor(x, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
gt = torch.as_tensor(g, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
params = {k: torch.as_tensor(v, dtype=torch.float32, device="cuda") for k, v in P.items()}
for _ in range(2):
    y, cache = neurons.forward(spec, params, xt)
    neurons.symbolic_backward(spec, params, cache, gt)
torch.cuda.synchronize()
print("ok")
