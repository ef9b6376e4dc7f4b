"""python tools/probe_coop_cluster.py: cooperative + 2-CTA cluster + PDL launches
(eager / graph), alone and next to a kernel holding some SMs."""
import ctypes
import os

import torch

here = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(here, "libprobe_coop_cluster.so"))
lib.probe_run.argtypes = [ctypes.c_int] * 6 + [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]
smem_kb = 150
mc = lib.probe_max_clusters(smem_kb)
print("max co-resident 2-CTA clusters at", smem_kb, "KB:", mc)
out = torch.zeros(4 * 148, dtype=torch.int32, device="cuda")
for clusters in (40, mc):
    for coop in (0, 1):
        for pdl in (0, 1):
            for graph in (0, 1):
                for busy in (0, 64):
                    if not coop and busy and clusters == mc:
                        continue  # would hang without the co-residency guarantee
                    ms = ctypes.c_float(0)
                    rc = lib.probe_run(clusters, smem_kb, coop, pdl, graph, busy, out.data_ptr(), ctypes.byref(ms))
                    o = out.cpu()
                    ok = rc == 0 and bool((o[2 * clusters:4 * clusters] == 2 * clusters).all())
                    print(f"clusters={clusters} coop={coop} pdl={pdl} graph={graph} busy={busy}: rc={rc} "
                          f"ok={ok} ms={ms.value:.3f}", flush=True)
