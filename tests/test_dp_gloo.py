"""Data-parallel gradient exchange on CPU: world_size 2 over gloo.

The bucketed all-reduce (paper_2204_01701_b200.dp) must leave every rank with
the mean of the per-rank gradients -- the DP parity oracle of SURVEY.md §8(e)
(mean over shards of per-shard gradients) -- across several buckets, and the
optimizer must be the reference sgd_step (trainer.py:50-61).
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _model():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(8, 32), torch.nn.ReLU(), torch.nn.Linear(32, 16),
                               torch.nn.ReLU(), torch.nn.Linear(16, 4))


def _data(rank):
    g = torch.Generator().manual_seed(100 + rank)
    return torch.randn(6, 8, generator=g), torch.randint(0, 4, (6,), generator=g)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2204_01701_b200.dp import BucketedAllReduce, broadcast_module
    m = _model()
    if rank == 1:  # a diverged replica is reset to rank 0's weights
        with torch.no_grad():
            for p in m.parameters():
                p.add_(1.0)
    broadcast_module(m)
    red = BucketedAllReduce(m.parameters(), bucket_mb=0.001)  # ~260 floats: several buckets
    assert len(red.buckets) >= 3
    for step in range(2):
        red.reset()
        x, y = _data(rank + 10 * step)
        loss = torch.nn.functional.cross_entropy(m(x), y)
        loss.backward()
        red.finish()
        if step == 0:
            out[rank] = [p.grad.detach().clone() for p in m.parameters()]
    dist.destroy_process_group()


def test_bucketed_allreduce_is_rank_mean():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    # oracle: mean over ranks of single-process gradients
    ref = None
    for r in range(world):
        m = _model()
        x, y = _data(r)
        torch.nn.functional.cross_entropy(m(x), y).backward()
        g = [p.grad.detach().clone() for p in m.parameters()]
        ref = g if ref is None else [a + b for a, b in zip(ref, g)]
    ref = [a / world for a in ref]
    for r in range(world):
        for a, b in zip(out[r], ref):
            assert torch.allclose(a, b, rtol=1e-5, atol=1e-6)


def test_single_process_reducer_accumulates_into_buckets():
    from paper_2204_01701_b200.dp import BucketedAllReduce
    m = _model()
    red = BucketedAllReduce(m.parameters(), bucket_mb=0.001)
    x, y = _data(0)
    torch.nn.functional.cross_entropy(m(x), y).backward()
    red.finish()
    flat_total = sum(f.numel() for f, _ in red.buckets)
    # every view starts 128-B aligned: the buckets hold the parameters plus < 32
    # padding elements each
    n = sum(p.numel() for p in m.parameters())
    assert n <= flat_total < n + 32 * len(list(m.parameters()))
    for flat, ps in red.buckets:  # offsets within the bucket (CUDA buffers themselves are 256-B aligned)
        for p in ps:
            assert (p.grad.data_ptr() - flat.data_ptr()) % 128 == 0
    # grads live in the buckets (views), so the bucket sums equal the grad sums
    assert torch.isclose(sum(f.sum() for f, _ in red.buckets),
                         sum(p.grad.sum() for p in m.parameters()))
    m2 = _model()
    torch.nn.functional.cross_entropy(m2(x), y).backward()
    for p, q in zip(m.parameters(), m2.parameters()):
        assert torch.allclose(p.grad, q.grad)


def test_sgd_matches_reference_sgd_step():
    """v <- m v + g + wd p ; p <- p - lr v  (reference trainer.py:50-61)."""
    from paper_2204_01701_b200.dp import sgd
    torch.manual_seed(1)
    p = torch.nn.Parameter(torch.randn(5))
    opt = sgd([p], lr=0.1)
    p_ref = p.detach().clone()
    v = None
    for it in range(3):
        g = torch.randn(5)
        p.grad = g.clone()
        opt.step()
        upd = g + 5e-4 * p_ref
        v = upd if v is None else 0.9 * v + upd
        p_ref = p_ref - 0.1 * v
        assert torch.allclose(p.detach(), p_ref, atol=1e-6)


def test_direct_gradient_sink_reports_each_parameter_once():
    """A function that writes its weight gradient straight into the bucket view
    (dp.take_grad) and returns None: the parameter is reported once (ready(),
    not again by the post-accumulate hook, which still fires), every bucket's
    counter reaches exactly zero, and the gradients equal autograd's."""
    from paper_2204_01701_b200.dp import BucketedAllReduce, grad_ready, take_grad

    class SinkLinear(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x, w, b):
            ctx.save_for_backward(x)
            ctx.w, ctx.b = w, b
            return x @ w.t() + b

        @staticmethod
        def backward(ctx, g):
            (x,) = ctx.saved_tensors
            out = []
            for p, grad in ((ctx.w, g.t() @ x), (ctx.b, g.sum(0))):
                t = take_grad(p)
                if t is None:
                    out.append(grad)
                else:
                    t.copy_(grad)
                    grad_ready(p)
                    out.append(None)
            return (g @ ctx.w, *out)

    torch.manual_seed(0)
    l1, l2 = torch.nn.Linear(5, 4), torch.nn.Linear(4, 3)
    ref1, ref2 = torch.nn.Linear(5, 4), torch.nn.Linear(4, 3)
    ref1.load_state_dict(l1.state_dict())
    ref2.load_state_dict(l2.state_dict())
    params = list(l1.parameters()) + list(l2.parameters())
    red = BucketedAllReduce(params, bucket_mb=4e-5)  # several buckets
    assert len(red.buckets) >= 2
    x = torch.randn(6, 5)
    for _ in range(2):  # the counters re-arm on reset()
        red.reset()
        h = SinkLinear.apply(x, l1.weight, l1.bias)
        y = l2(torch.relu(h))  # l2 through autograd (AccumulateGrad + hook)
        y.square().sum().backward()
        assert red.pending == [0] * len(red.buckets)
        red.finish()
    for r in (ref1, ref2):
        r.zero_grad()
    ref2(torch.relu(ref1(x))).square().sum().backward()
    for p, q in zip(params, list(ref1.parameters()) + list(ref2.parameters())):
        assert torch.allclose(p.grad, q.grad, atol=1e-6)
