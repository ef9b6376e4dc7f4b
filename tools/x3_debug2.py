import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import _lib, neurons
from paper_2204_01701_b200.spec import QuadraticLayerSpec
n, c, f, hw = 2, 64, 64, 32
for fam in ("first_order", "proposed"):
    spec = QuadraticLayerSpec(kind="conv", family=fam, in_dim=c, out_dim=f, kernel=3, stride=1, pad=1)
    x, P, g = Q.synthetic_layer(fam, "conv", n, c, f, hw, hw, 3, 1, 1, seed=0)
    dev = torch.device("cuda")
    xt = torch.as_tensor(x, device=dev).float().contiguous(memory_format=torch.channels_last)
    params = {r: torch.as_tensor(v, dtype=torch.float32, device=dev) for r, v in P.items()}
    y3 = neurons.forward(spec, params, xt)[0].double().cpu().numpy()
    y0 = neurons.forward(spec, params, xt, flags=_lib.FLAG_FORCE_SIMT)[0].double().cpu().numpy()
    print(fam, "path", neurons.device_path(spec, x.shape, torch.float32))
    for h in range(0, 12):
        errs = [np.abs(y3[0, :, h, :] - y0[0, :, hh, :]).max() for hh in range(hw)]
        best = int(np.argmin(errs))
        print(" h", h, "err same", f"{errs[h]:.2e}", "best match h", best, f"{errs[best]:.2e}",
              "x3 absmax", f"{np.abs(y3[0, :, h, :]).max():.2e}")
