import ctypes, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libprobe_mma.so"))
lib.mma_rate_run.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 5
out = torch.zeros(2, dtype=torch.int64, device="cuda")
torch.zeros(1, device="cuda")
for cg, n, u in [(1,64,4),(1,128,4),(1,192,4),(1,256,4),(2,64,4),(2,128,4),(2,192,4),(2,256,4),(1,64,16),(2,64,16),(2,192,16)]:
    for grid in (cg, 148):
        iters = 1024
        st = lib.mma_rate_run(out.data_ptr(), cg, n, u, iters, grid)
        issue, total = out.tolist()
        ideal = (256 if cg == 2 else 128) * n / (256 * cg)
        print(f"cg={cg} N={n:3d} unroll={u:2d} grid={grid:3d} st={st} issue/MMA={issue/iters:7.1f} total/MMA={total/iters:7.1f} cyc  (floor {ideal:.0f})", flush=True)
