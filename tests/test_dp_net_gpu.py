"""Data-parallel training of the real QuadraNet step: world size 2 over gloo.

Two ranks (processes) each run the full QuadraVGG-16 / QuadraResNet-18
training step on their own batch shard with the device kernels -- quadratic
layers, fused BN, max pool, fused SGD + pack -- and exchange gradients through
``dp.BucketedAllReduce`` (post-accumulate hooks, bucketed AVG all-reduce).
DP parity oracle: every rank's gradients equal the mean of
the per-shard gradients of single-process steps from the same start state,
and after one ``QuadSGD`` step (trainer.py:50-61 semantics) every replica
holds the same parameters, equal to the single-process update with the mean
gradient.

Both ranks share the one GPU of the box; their kernels never wait on each
other (the exchange is gloo, on the host), and the in-kernel grid barrier of
the wgrad fold is switched off in the workers (QD_W3_NOFOLD=1) so nothing
spins across the two contexts. The NCCL transport of the same reducer is the
bench's multi-GPU path.
"""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = {"qvgg16": ("QuadraVGG16", 10, 4, 32), "qresnet18": ("QuadraResNet18", 1000, 2, 64)}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _build(net):
    from paper_2204_01701_b200 import qnets
    builder, classes, _, _ = CASES[net]
    torch.manual_seed(5)
    return getattr(qnets, builder)(num_classes=classes).cuda().to(memory_format=torch.channels_last)


def _shard(net, rank):
    _, classes, batch, hw = CASES[net]
    g = torch.Generator(device="cuda").manual_seed(100 + rank)
    x = torch.randn(batch, 3, hw, hw, device="cuda", generator=g).bfloat16().contiguous(
        memory_format=torch.channels_last)
    return x, torch.randint(0, classes, (batch,), device="cuda", generator=g)


def _step(model, red, opt, x, y):
    red.reset()
    with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
        loss = torch.nn.functional.cross_entropy(model(x), y)
    loss.backward()
    red.finish()
    grads = {n: p.grad.detach().float().cpu().clone() for n, p in model.named_parameters()}
    opt.step()
    torch.cuda.synchronize()
    return grads, {n: p.detach().float().cpu().clone() for n, p in model.named_parameters()}


def _worker(rank, world, port, net, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["QD_W3_NOFOLD"] = "1"
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_01701_b200.dp import BucketedAllReduce, broadcast_module
    from paper_2204_01701_b200.optim import QuadSGD
    model = _build(net)
    if rank == 1:  # a diverged replica is reset to rank 0's start state
        with torch.no_grad():
            for p in model.parameters():
                p.mul_(1.5)
    broadcast_module(model)
    opt = QuadSGD(model, lr=0.05)
    red = BucketedAllReduce(model.parameters(), bucket_mb=8.0)
    x, y = _shard(net, rank)
    grads, params = _step(model, red, opt, x, y)
    out[rank] = (grads, params, len(red.buckets))
    dist.destroy_process_group()


@pytest.mark.parametrize("net", sorted(CASES))
def test_dp_world2_matches_mean_of_shards(net):
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, port, net, out), nprocs=world, join=True, start_method="spawn")
    assert out[0][2] >= 2  # several buckets in flight
    # oracle: single-process steps per shard from the same start state, gradients averaged
    os.environ["QD_W3_NOFOLD"] = "1"
    try:
        from paper_2204_01701_b200.dp import BucketedAllReduce
        from paper_2204_01701_b200.optim import QuadSGD
        per = []
        for r in range(world):
            model = _build(net)
            red = BucketedAllReduce(model.parameters(), bucket_mb=8.0)
            g, _ = _step(model, red, QuadSGD(model, lr=0.05), *_shard(net, r))
            per.append(g)
        model = _build(net)
        start = {n: p.detach().float().cpu().clone() for n, p in model.named_parameters()}
    finally:
        del os.environ["QD_W3_NOFOLD"]
    mean = {n: (per[0][n] + per[1][n]) / 2 for n in per[0]}
    for r in range(world):
        grads, params, _ = out[r]
        for n in mean:
            assert torch.allclose(grads[n], mean[n], rtol=1e-5, atol=1e-7), (r, n)
            want = start[n] - 0.05 * (mean[n] + 5e-4 * start[n])
            assert torch.allclose(params[n], want, rtol=1e-5, atol=1e-6), (r, n)
    for n in mean:  # replicas identical
        assert torch.equal(out[0][1][n], out[1][1][n]), n
