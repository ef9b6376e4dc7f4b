"""python tools/tf32_peak.py: cuBLAS TF32 dense peak, measured like MEASURED_PEAKS.json's bf16
figure (8192^3 matmul, best of 10 with CUDA events; back to back for ~4 s = sustained)."""
import json
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a @ b
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
burst = 2 * n ** 3 / (best * 1e-3) / 1e12
t0 = time.time()
k = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        a @ b
    k += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sus = 2 * n ** 3 * k / (e0.elapsed_time(e1) * 1e-3) / 1e12
print(json.dumps({"tf32_tflops": burst, "tf32_tflops_sustained": sus, "how": "torch.matmul fp32 with TF32 "
                  "allowed, 8192^3: best of 10 (burst) and back to back for 4 s (sustained)"}))
