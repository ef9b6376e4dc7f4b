"""Run the descriptor-shift probe (tools/probe_desc.cu) and print which
(shift, base_offset) combinations reproduce the shifted GEMM exactly."""
import ctypes
import os
import sys

import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libprobe.so"))
lib.probe_run.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3
torch.manual_seed(0)
dev = "cuda"
res = {}
for mode in (0, 1):
    if mode == 0:
        A = torch.randn(256, 64, device=dev).bfloat16()
        B = torch.randn(64, 64, device=dev).bfloat16()
    else:
        A = torch.randn(256, 128, device=dev).bfloat16()
        B = torch.randn(256, 64, device=dev).bfloat16()
    out = torch.empty(128, 64, device=dev)
    for shift in (0, 1, 2, 3, 5, 7, 8, 9, 35, 70):
        for bo in sorted({0, shift % 8}):
            out.zero_()
            st = lib.probe_run(A.data_ptr(), B.data_ptr(), out.data_ptr(), mode, shift, bo)
            if mode == 0:
                ref = A[shift:shift + 128].float() @ B.float().T
            else:
                ref = A[shift:shift + 64].float().T @ B[:64].float()
            err = ((out - ref).abs().max() / ref.abs().max()).item()
            ok = err < 1e-3
            res[(mode, shift, bo)] = ok
            print(f"mode={mode} shift={shift:3d} base_off={bo} status={st} rel_err={err:.2e} {'OK' if ok else 'BAD'}")
sys.stdout.flush()
