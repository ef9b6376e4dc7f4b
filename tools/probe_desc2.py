"""Modes 2/3 of tools/probe_desc.cu: overlapping MN-major atoms (LBO < atom) and
TMA SW128 loads into 128-B (not 1024-B) aligned destinations."""
import ctypes, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libprobe.so"))
lib.probe_run.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3
torch.manual_seed(0)
A = torch.randn(256, 64, device="cuda").bfloat16()
B = torch.randn(256, 64, device="cuda").bfloat16()
out = torch.empty(128, 64, device="cuda")
for shift in (0, 3):
    for lbo_rows in (1, 2, 7, 8, 34, 36):
        out.zero_()
        st = lib.probe_run(A.data_ptr(), B.data_ptr(), out.data_ptr(), 2, shift, lbo_rows)
        top = A[shift:shift + 64].float().T @ B[:64].float()
        bot = A[shift + lbo_rows:shift + lbo_rows + 64].float().T @ B[:64].float()
        ref = torch.cat([top, bot])
        err = ((out - ref).abs().max() / ref.abs().max()).item()
        print(f"mode=2 shift={shift} lbo_rows={lbo_rows} status={st} err={err:.2e} {'OK' if err < 1e-3 else 'BAD'}", flush=True)
A3 = torch.randn(192, 64, device="cuda").bfloat16()
B3 = torch.randn(64, 64, device="cuda").bfloat16()
for d in (0, 1, 2, 5, 7):
    for shift in (0, 1, 6):
        out.zero_()
        st = lib.probe_run(A3.data_ptr(), B3.data_ptr(), out.data_ptr(), 3, shift, d)
        ref = A3[shift:shift + 128].float() @ B3.float().T
        err = ((out - ref).abs().max() / ref.abs().max()).item()
        print(f"mode=3 dst_off_rows={d} shift={shift} status={st} err={err:.2e} {'OK' if err < 1e-3 else 'BAD'}", flush=True)
