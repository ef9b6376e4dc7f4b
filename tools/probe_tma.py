"""TMA throughput for conv box shapes (tools/probe_tma.cu)."""
import ctypes, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libprobe_tma.so"))
lib.tma_probe_run.restype = ctypes.c_float
lib.tma_probe_run.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 11
N, H, W = 128, 32, 32
x = torch.randn(N, H, W, 64, device="cuda").bfloat16()
cases = [
    ("v1 tap box 32x4 w0=0", 0, 32, 4, 0, 0),
    ("v1 tap box 32x4 w0=-1 (OOB col)", 0, 32, 4, -1, 0),
    ("halo 34x7 w0=-1 (2 OOB cols)", 0, 34, 7, -1, 0),
    ("halo 32x7 w0=0", 0, 32, 7, 0, 0),
    ("box 32x8 w0=0", 0, 32, 8, 0, 0),
    ("2D 238 rows", 1, 0, 0, 0, 238),
    ("2D 128 rows", 1, 0, 0, 0, 128),
    ("2D 256 rows", 1, 0, 0, 0, 256),
]
for stages in (2, 4, 6):
    for name, mode, bw, bh, w0, rows in cases:
        boxb = (bw * bh if mode == 0 else rows) * 128
        slot = (boxb + 1023) // 1024 * 1024
        if stages * slot > 200 * 1024:
            continue
        iters = 200
        for ctas in (148,):
            ms = lib.tma_probe_run(x.data_ptr(), N, H, W, mode, bw, bh, w0, rows, stages, iters, ctas)
            gbs = ctas * iters * boxb / (ms * 1e-3) / 1e9 if ms > 0 else -1
            print(f"stages={stages} {name:34s} box={boxb/1024:5.1f}KB  {ms*1e3:8.1f}us  {gbs:8.0f} GB/s", flush=True)
