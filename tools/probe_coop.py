"""python tools/probe_coop.py: cooperative launch (grid.sync) eager and inside graph capture."""
import ctypes, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libprobe_coop.so"))
lib.probe_coop.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
mb = lib.probe_coop_maxblocks()
print("max co-resident blocks", mb)
n = 1 << 24
x = torch.ones(n, device="cuda")
part = torch.zeros(mb, device="cuda")
out = torch.zeros(1, device="cuda")
st = torch.cuda.current_stream().cuda_stream
print("eager rc", lib.probe_coop(x.data_ptr(), part.data_ptr(), out.data_ptr(), n, mb, st))
torch.cuda.synchronize()
print("eager sum", out.item(), "expect", n)
out.zero_()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g):
        rc = lib.probe_coop(x.data_ptr(), part.data_ptr(), out.data_ptr(), n, mb, torch.cuda.current_stream().cuda_stream)
print("capture rc", rc)
g.replay()
torch.cuda.synchronize()
print("graph sum", out.item())
