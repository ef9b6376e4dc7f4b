"""fp32 QuadConvBN (fused BN backward -> D given -> x3 path) vs an fp64 composition."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import net_oracle as NO
from paper_2204_01701_b200.bn import QuadConvBN
from paper_2204_01701_b200.nn import QuadConv2d
from paper_2204_01701_b200 import neurons
torch.manual_seed(0)
for relu in (True, False):
  for (n, c, f, hw) in [(4, 64, 64, 16), (8, 64, 128, 8), (8, 128, 128, 4)]:
    layer = QuadConv2d(c, f, 3, 1, 1, device="cuda", compute_dtype=torch.float32)
    mod = QuadConvBN(layer, relu=relu)
    with torch.no_grad():
        mod.weight.uniform_(0.5, 1.5); mod.bias.uniform_(-0.2, 0.2)
        for r in ("ba", "bb", "bc"): getattr(layer, r).uniform_(-0.1, 0.1)
    x = torch.randn(n, c, hw, hw, device="cuda").contiguous(memory_format=torch.channels_last)
    gz = torch.randn(n, f, hw, hw, device="cuda")
    z = mod(x.requires_grad_(True))
    z.backward(gz)
    P = {r: getattr(layer, r).detach().double().cpu().requires_grad_(True) for r in ("Wa", "Wb", "Wc", "ba", "bb", "bc")}
    gam = mod.weight.detach().double().cpu().requires_grad_(True); bet = mod.bias.detach().double().cpu().requires_grad_(True)
    xx = x.detach().double().cpu().requires_grad_(True)
    zr = NO.batchnorm(NO.quad_conv(xx, P, "", "proposed", 1, 1), gam, bet)
    if relu: zr = zr * (z.detach().cpu() > 0).double()
    zr.backward(gz.double().cpu())
    fro = lambda a, b: float((a.detach().double().cpu() - b.detach().double().cpu()).norm() / b.norm())
    errs = {"z": fro(z, zr), "dx": fro(x.grad, xx.grad), "gamma": fro(mod.weight.grad, gam.grad), "beta": fro(mod.bias.grad, bet.grad)}
    errs.update({r: fro(getattr(layer, r).grad, P[r].grad) for r in ("Wa", "Wb", "Wc", "ba", "bb")})
    print(relu, n, c, f, hw, "path", neurons.device_path(layer.spec, x.shape, torch.float32), "fused", mod.fused(x),
          {k: f"{v:.1e}" for k, v in errs.items()}, flush=True)
