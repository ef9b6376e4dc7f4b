"""python tools/x3_debug.py: fp32 split tensor-core path vs the FFMA path on the C2 geometry at growing N."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import quadra_oracle as Q
from paper_2204_01701_b200 import _lib, neurons
from paper_2204_01701_b200.spec import QuadraticLayerSpec

for (n, c, f, hw) in [(2, 64, 64, 32), (8, 64, 64, 32), (32, 64, 64, 32), (64, 64, 64, 32), (128, 64, 64, 32),
                      (16, 64, 64, 56), (4, 128, 128, 28)]:
    spec = QuadraticLayerSpec(kind="conv", family="proposed", in_dim=c, out_dim=f, kernel=3, stride=1, pad=1)
    x, P, g = Q.synthetic_layer("proposed", "conv", n, c, f, hw, hw, 3, 1, 1, seed=0, random_bias=True)
    dev = torch.device("cuda")
    xt = torch.as_tensor(x, device=dev).float().contiguous(memory_format=torch.channels_last)
    gt = torch.as_tensor(g, device=dev).float().contiguous(memory_format=torch.channels_last)
    params = {r: torch.as_tensor(v, dtype=torch.float32, device=dev) for r, v in P.items()}
    out = []
    for flags in (0, _lib.FLAG_FORCE_SIMT):
        y, cache = neurons.forward(spec, params, xt, flags=flags)
        grads, dx = neurons.symbolic_backward(spec, params, cache, gt)
        torch.cuda.synchronize()
        out.append((y.double().cpu().numpy(), cache.a.double().cpu().numpy(), dx.double().cpu().numpy(),
                    {k: v.double().cpu().numpy() for k, v in grads.items()}))
    path = neurons.device_path(spec, x.shape, torch.float32)
    e = {"y": Q.rel_err(out[0][0], out[1][0]), "a": Q.rel_err(out[0][1], out[1][1]),
         "dx": Q.rel_err(out[0][2], out[1][2])}
    e.update({k: Q.rel_err(out[0][3][k], out[1][3][k]) for k in out[0][3]})
    import numpy as np
    bad = np.argwhere(np.abs(out[0][0] - out[1][0]) > 1e-3 * np.abs(out[1][0]).max())
    print(n, c, f, hw, "path", path, {k: f"{v:.1e}" for k, v in e.items()}, "bad y elems", len(bad),
          bad[:3].tolist(), flush=True)
