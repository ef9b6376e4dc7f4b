"""Does an NCCL all-reduce issued from an autograd hook capture into a CUDA graph?
(world_size 1 NCCL group; the bucket hooks are forced on). python tools/nccl_graph_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
from paper_2204_01701_b200 import qnets
from paper_2204_01701_b200.dp import BucketedAllReduce
from paper_2204_01701_b200.graphstep import GraphedStep
from paper_2204_01701_b200.optim import QuadSGD
torch.manual_seed(0)
m = qnets.QuadraVGG16(10).cuda().to(memory_format=torch.channels_last)
opt = QuadSGD(m, lr=0.01)
red = BucketedAllReduce(m.parameters(), bucket_mb=4.0)
red.world = 2  # force the hooks to issue their NCCL all-reduces (the group has one rank)
x = torch.randn(32, 3, 32, 32, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
y = torch.randint(0, 10, (32,), device="cuda")


def step(xb, yb):
    red.reset()
    with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
        loss = torch.nn.functional.cross_entropy(m(xb), yb)
    loss.backward()
    red.finish()
    opt.step()
    return loss


gs = GraphedStep(step, x, y)
l = [float(gs()) for _ in range(5)]
print("captured with NCCL all-reduces:", len(red.buckets), "buckets; losses", [round(v, 4) for v in l])
dist.destroy_process_group()
