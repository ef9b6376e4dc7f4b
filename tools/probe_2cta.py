"""Run tools/probe_2cta.cu: which B distribution does cta_group::2 expect?"""
import ctypes, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libprobe2.so"))
lib.probe2_run.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int]
torch.manual_seed(0)
A = torch.randn(256, 64, device="cuda").bfloat16()
B = torch.randn(64, 64, device="cuda").bfloat16()
ref = A.float() @ B.float().T
for variant, name in ((0, "split"), (1, "full")):
    out = torch.zeros(256, 64, device="cuda")
    st = lib.probe2_run(A.data_ptr(), B.data_ptr(), out.data_ptr(), variant)
    err = ((out - ref).abs().max() / ref.abs().max()).item()
    # also test: does each CTA's half use only its own 32 B rows for all 64 cols?
    print(f"variant={name} status={st} rel_err={err:.2e} {'OK' if err < 1e-3 else 'BAD'}", flush=True)
    if err >= 1e-3:
        for half in (0, 1):
            blk = out[128 * half:128 * half + 128]
            for nb in (0, 1):
                sub = blk[:, 32 * nb:32 * nb + 32]
                r = ref[128 * half:128 * half + 128, 32 * nb:32 * nb + 32]
                e = ((sub - r).abs().max() / r.abs().max()).item()
                print(f"   half={half} ncols={32*nb}-{32*nb+31} err={e:.2e}")
