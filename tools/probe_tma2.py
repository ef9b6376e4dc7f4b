"""conv2-pattern TMA pipeline rate (tools/probe_tma2.cu). Build: see tools/build_probe2.sh"""
import ctypes, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libprobe_tma2.so"))
lib.probe2_run.restype = ctypes.c_float
lib.probe2_run.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 10 + [ctypes.c_void_p]
cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
for (N, H, W, bw, bh, w0, label) in [(128, 32, 32, 34, 7, -1, "C2 halo 34x7"), (128, 32, 32, 32, 7, 0, "in-bounds 32x7"),
                                      (512, 64, 64, 64, 3, 0, "big tensor 64x3 (cold)")]:
    x = torch.randn(N, H, W, 64, device="cuda").bfloat16()
    for mode in (0, 1, 2):
        for slots in (1, 2, 3, 6):
            if slots * ((bw * bh * 128 + 1023) // 1024 * 1024) > 200 * 1024:
                continue
            iters = 64
            ms = lib.probe2_run(x.data_ptr(), N, H, W, mode, bw, bh, w0, slots, iters, 74, cyc.data_ptr())
            per = ms * 1e3 / iters
            print(f"{label:24s} mode={mode} slots={slots}: {ms*1e3:7.1f} us total, {per*1e3:6.0f} ns/box/CTA, "
                  f"cyc/box {int(cyc.item())/iters:6.0f}, {148*iters*bw*bh*128/(ms*1e-3)/1e9:7.0f} GB/s", flush=True)
