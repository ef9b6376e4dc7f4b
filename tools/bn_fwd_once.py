"""One BN forward (+ backward) at a given shape, for ncu captures (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01701_b200.bn import BNAct2d

n, c, hw = (int(v) for v in sys.argv[1:4])
x = torch.randn(n, c, hw, hw, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
m = BNAct2d(c, relu=True).cuda()
for _ in range(3):
    x1 = x.detach().requires_grad_(True)
    z = m(x1)
    z.backward(torch.ones_like(z))
torch.cuda.synchronize()
