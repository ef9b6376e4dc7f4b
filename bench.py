#!/usr/bin/env python
"""Benchmark of the quadratic-layer hot path (BASELINE.json metric).

Default workload (N=1): BASELINE config 2 -- one quadratic conv layer
(proposed neuron), NCHW 128x64x32x32 -> 64, 3x3/s1/p1, bf16, forward +
backward. A "step" = pack weights + forward + backward (weight, bias and
input gradients) over one batch. Metric: algorithmic TFLOP/s
(9 GEMMs x 2*M*K*N: 86.97 GFLOP per step).

Multi-GPU (torchrun, one rank per GPU): weak scaling, every rank runs its own
batch-128 step and the weight/bias gradients are all-reduced (mean) over NCCL
each step -- the one real exchange of data-parallel training.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c5_64x56|...]

``--impl reference`` times the reference algorithm on the host CPU (the
oracle port of the reference's numpy path; the reference is pure Python and
is not installable on the GPU box) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (family, kind, N, C, F, H, W, r, s, p, dtype)
    "c2": ("proposed", "conv", 128, 64, 64, 32, 32, 3, 1, 1, "bf16"),
    "c2_fp32": ("proposed", "conv", 128, 64, 64, 32, 32, 3, 1, 1, "fp32"),
    "c1": ("proposed", "fc", 256, 512, 512, 1, 1, 1, 1, 0, "fp32"),
    "x3_128x28": ("proposed", "conv", 64, 128, 128, 28, 28, 3, 1, 1, "fp32"),
    "x3_64x56": ("proposed", "conv", 64, 64, 64, 56, 56, 3, 1, 1, "fp32"),
    "c5_proposed_64x56": ("proposed", "conv", 64, 64, 64, 56, 56, 3, 1, 1, "bf16"),
    "c5_proposed_128x28": ("proposed", "conv", 64, 128, 128, 28, 28, 3, 1, 1, "bf16"),
    "c5_proposed_256x14": ("proposed", "conv", 64, 256, 256, 14, 14, 3, 1, 1, "bf16"),
    "c5_proposed_512x7": ("proposed", "conv", 64, 512, 512, 7, 7, 3, 1, 1, "bf16"),
    "c5_t4_64x56": ("t4", "conv", 64, 64, 64, 56, 56, 3, 1, 1, "bf16"),
    "c5_t2lin_64x56": ("t2_linear", "conv", 64, 64, 64, 56, 56, 3, 1, 1, "bf16"),
    "c5_t4_512x7": ("t4", "conv", 64, 512, 512, 7, 7, 3, 1, 1, "bf16"),
    "c5_t2lin_512x7": ("t2_linear", "conv", 64, 512, 512, 7, 7, 3, 1, 1, "bf16"),
    # families beyond the BASELINE sweep
    "c5_t3_64x56": ("t3", "conv", 64, 64, 64, 56, 56, 3, 1, 1, "bf16"),
    "c5_t2and4_64x56": ("t2and4", "conv", 64, 64, 64, 56, 56, 3, 1, 1, "bf16"),
    "dw_proposed_256x28": ("proposed", "dwconv", 64, 256, 256, 28, 28, 3, 1, 1, "bf16"),
    # QuadraVGG-16 layer shapes at its bench batch (per-layer profiling)
    # QuadraResNet-18 quadratic layers (batch 128; stride-2 = first conv of stages 2-4)
    "r18_64x56": ("proposed", "conv", 128, 64, 64, 56, 56, 3, 1, 1, "bf16"),
    "r18_s2_64x56": ("proposed", "conv", 128, 64, 128, 56, 56, 3, 2, 1, "bf16"),
    "r18_128x28": ("proposed", "conv", 128, 128, 128, 28, 28, 3, 1, 1, "bf16"),
    "r18_s2_128x28": ("proposed", "conv", 128, 128, 256, 28, 28, 3, 2, 1, "bf16"),
    "r18_256x14": ("proposed", "conv", 128, 256, 256, 14, 14, 3, 1, 1, "bf16"),
    "r18_s2_256x14": ("proposed", "conv", 128, 256, 512, 14, 14, 3, 2, 1, "bf16"),
    "r18_512x7": ("proposed", "conv", 128, 512, 512, 7, 7, 3, 1, 1, "bf16"),
    "vgg_64x32": ("proposed", "conv", 256, 64, 64, 32, 32, 3, 1, 1, "bf16"),
    "vgg_128x16": ("proposed", "conv", 256, 128, 128, 16, 16, 3, 1, 1, "bf16"),
    "vgg_256x8": ("proposed", "conv", 256, 256, 256, 8, 8, 3, 1, 1, "bf16"),
    "vgg_512x4": ("proposed", "conv", 256, 512, 512, 4, 4, 3, 1, 1, "bf16"),
    "vgg_512x2": ("proposed", "conv", 256, 512, 512, 2, 2, 3, 1, 1, "bf16"),
}
METRIC = "quadratic_conv_fwd_bwd_tflops"
TF32_PEAK = 720.9  # cuBLAS TF32 8192^3 burst on this pool's B200 (tools/tf32_peak.py, profiles/r2_tf32_peak.json)
L2_NOTE = ("flushed between timed steps (untimed): 256 MiB write, then a 256 MiB read so the "
           "step starts from a cold, clean L2 (no dirty-line write-back billed to the step)")


def flush_l2(buf, i):
    """Evict L2 between timed steps: write a buffer 2x larger than L2, then read it
    back (the read leaves clean lines; the write-back of the flush happens here)."""
    buf.fill_(i & 0xFF)
    buf.view(-1, 4096).amax(dim=1, keepdim=False).sum()


def pipelined_e2e(k, h2d, compute, d2h):
    """ms per step of k end-to-end steps through host memory: h2d(b) fills device
    input set b on a copy-in stream, compute(b) runs on the current stream and
    returns its result tensors, d2h(outs) copies them to pinned host memory on a
    copy-out stream. Inputs are double-buffered, so step i+1's H2D overlaps step
    i's compute and step i-1's D2H (PCIe is full duplex) -- a prefetching input
    pipeline; every step still moves its own inputs and results. Timed with CUDA
    events on the compute stream around all k steps (pipeline fill included)."""
    import torch
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    in_done = [torch.cuda.Event(), torch.cuda.Event()]
    freed = [torch.cuda.Event(), torch.cuda.Event()]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(comp)
    s_in.wait_stream(comp)
    s_out.wait_stream(comp)

    def issue_in(i):
        b = i % 2
        with torch.cuda.stream(s_in):
            if i >= 2:
                s_in.wait_event(freed[b])  # compute i-2 is done with set b
            h2d(b)
            in_done[b].record(s_in)

    issue_in(0)
    for i in range(k):
        b = i % 2
        if i + 1 < k:
            issue_in(i + 1)
        comp.wait_event(in_done[b])
        outs = compute(b)
        freed[b].record(comp)
        done = torch.cuda.Event()
        done.record(comp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(done)
            for t_ in outs:
                t_.record_stream(s_out)
            d2h(outs)
    comp.wait_stream(s_out)
    e1.record(comp)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return {"bf16": pk["bf16_tflops"], "bf16_sustained": pk["bf16_tflops_sustained"],
                "hbm": pk["hbm_gbs"], "src": "measured"}
    except Exception:  # noqa: BLE001
        return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "src": "fallback"}


def make_spec(wl):
    from paper_2204_01701_b200.spec import QuadraticLayerSpec
    fam, kind, n, c, f, h, w, r, s, p, _ = wl
    return QuadraticLayerSpec(kind=kind, family=fam, in_dim=c, out_dim=f, kernel=r, stride=s,
                              pad=p)


def flops_of(wl, n=None):
    from paper_2204_01701_b200.spec import gemm_flops
    fam, kind, n0, c, f, h, w, r, s, p, _ = wl
    return gemm_flops(make_spec(wl), n if n is not None else n0, h, w)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock + throttle reasons polled through NVML every ~2 ms on a thread
    (nvidia-smi's 200 ms floor cannot see a millisecond-long timed region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index, period=0.002):
        self.index = index
        self.period = period
        self.samples = []  # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self._stop = threading.Event()
        self.thread = None
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001
            self.nvml = None
        return self

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:  # noqa: BLE001
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((mhz, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self.thread is not None:
            self.thread.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        reasons = set()
        for _, rs in self.samples:
            for nm, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median([m for m, _ in self.samples]), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def sampled_clocks(local, timed_clk, replay, ms_step, world=1, seconds=0.4):
    """Clock line for the JSON: the timed region's samples when there are enough,
    else (timed region of a few ms) a sustained replay of the same step right after.
    The replay count is derived from the rank-max step time, so every rank runs the
    same number of steps (they may contain collectives)."""
    import torch
    tc = timed_clk.summary()
    if world == 1 and tc["samples"] >= 5:
        tc["window"] = "timed region"
        return tc
    iters = max(20, int(seconds * 1e3 / max(ms_step, 1e-3)))
    with ClockSampler(local) as clk:
        for i in range(iters):
            replay()
            if i % 50 == 49:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
    sc = clk.summary()
    sc["window"] = f"sustained replay of {iters} steps right after the timed region " \
                   f"(timed region: {tc['samples']} samples, median {tc['sm_mhz']} MHz)"
    return sc


# ---------------------------------------------------------------------------
# CPU side: the reference algorithm (oracle port of the reference's numpy path)
# ---------------------------------------------------------------------------
def cpu_sample(wl, batch, reps):
    """Time reference forward + symbolic_backward (fp64 numpy, all host
    threads) on `batch` samples; returns (best seconds, flops)."""
    from oracle import quadra_oracle as Q
    fam, kind, n, c, f, h, w, r, s, p, _ = wl
    x, P, g = Q.synthetic_layer(fam, kind, batch, c, f, h, w, r, s, p, seed=0)
    geo = Q.Geometry(kind, r, s, p)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        y, a, b = Q.forward(fam, geo, P, x)
        Q.symbolic_backward(fam, geo, P, x, a, b, g)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, flops_of(wl, batch)


def cpu_batch_for(wl):
    """Bounded CPU sample: ~1-3 s per repetition on a few host cores."""
    fam, kind, n, c, f, h, w, r, s, p, _ = wl
    if kind == "fc":
        return n
    per_sample = flops_of(wl, 1)
    return max(1, min(n, int(6e9 // per_sample)))


def run_reference(args, wl, wl_name):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count()
    batch = cpu_batch_for(wl)
    times = []
    flops = flops_of(wl, batch)
    for i in range(args.warmup + args.steps):
        t, _ = cpu_sample(wl, batch, 1)
        if i >= args.warmup:
            times.append(t)
    mean = sum(times) / len(times)
    value = flops / mean / 1e12
    sample = (f"{wl_name} at batch {batch} of {wl[2]} (fp64 numpy/BLAS reference algorithm: "
              f"im2col + GEMM + col2im), mean of {args.steps} steps")
    # ms_per_step is the MEASURED time of one step of the bounded sample (batch
    # `step_batch`); value is its rate, which is linear in the batch (im2col, GEMM M
    # and col2im all scale with N)
    out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "impl": "reference",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": mean * 1e3, "step_batch": batch, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_of(wl, wl_name, args.gpus),
           "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                            "sample": sample},
           "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    nets = {}
    for net in args.nets:
        secs = [net_cpu_baseline(net) for _ in range(max(1, min(args.steps, 3)))]
        sec = sum(secs) / len(secs)
        nets[net] = {"metric": f"{net}_train_img_per_s", "value": 1.0 / sec, "unit": "img/s",
                     "ms_per_step": sec * 1e3, "step_batch": 1,
                     "sample": "reference algorithm fwd+bwd of every quadratic layer at batch 1, summed"}
    out["nets"] = nets
    print(json.dumps(out), flush=True)
    return 0


def config_of(wl, name, ngpu):
    fam, kind, n, c, f, h, w, r, s, p, dt = wl
    return {"workload": f"{name}: {fam} {kind} {n}x{c}x{h}x{w} -> {f}, k{r} s{s} p{p}, {dt}",
            "family": fam, "global_batch": n * ngpu, "per_gpu_batch": n,
            "parallelism": f"dp{ngpu}",
            "l2": L2_NOTE,
            "flops_per_step_per_gpu": flops_of(wl)}


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------
def _dist(world):
    """a process group is up: world > 1, or QD_DIST_FORCE=1 (dev: the NCCL path --
    process group, collectives, graph-captured bucket all-reduces -- exercised by
    a single-rank torchrun on one GPU)"""
    return world > 1 or os.environ.get("QD_DIST_FORCE") == "1"


def run_ours(args, wl, wl_name):
    import torch
    import torch.distributed as dist

    from paper_2204_01701_b200 import _lib, neurons

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if _dist(world):
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    fam, kind, n, c, f, h, w, r, s, p, dts = wl
    dt = torch.bfloat16 if dts == "bf16" else torch.float32
    spec = make_spec(wl)

    from oracle import quadra_oracle as Q  # seeded input generator only (not timed)
    x64, P64, g64 = Q.synthetic_layer(fam, kind, n, c, f, h, w, r, s, p, seed=rank)
    if rank:  # replicas share rank 0's weights; inputs are per-rank shards
        P64 = Q.synthetic_layer(fam, kind, 1, c, f, h, w, r, s, p, seed=0)[1]
    x = torch.as_tensor(x64, device=dev).to(dt)
    gy = torch.as_tensor(g64, device=dev).to(dt)
    if kind != "fc":
        x = x.contiguous(memory_format=torch.channels_last)
        gy = gy.contiguous(memory_format=torch.channels_last)
    params = {k_: torch.as_tensor(v, dtype=torch.float32, device=dev) for k_, v in P64.items()}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    # the layer's weight / bias gradients land in one flat fp32 buffer (the
    # library writes them there directly), so the data-parallel exchange is one
    # all-reduce with no gather copy; captured into the step's graph below
    gorder = [r_ for r_ in neurons.GRAD_ORDER[fam] if r_ in params]
    gflat = torch.zeros(sum(params[r_].numel() for r_ in gorder), dtype=torch.float32, device=dev)
    gviews, o_ = {}, 0
    for r_ in gorder:
        gviews[r_] = gflat[o_:o_ + params[r_].numel()].view(params[r_].shape)
        o_ += params[r_].numel()

    def compute(want_dx=True, want_dw=True, out=gviews):
        y, cache = neurons.forward(spec, params, x, dtype=dt)
        grads, dx = neurons.symbolic_backward(spec, params, cache, gy, want_dx=want_dx,
                                              want_dw=want_dw, out=out)
        return y, grads, dx

    def exchange(grads):
        # the one data-parallel exchange: rank mean of dW / db
        if _dist(world):
            if all(grads[r_] is gviews[r_] for r_ in gorder if r_ in grads):
                dist.all_reduce(gflat, op=dist.ReduceOp.AVG)
            else:
                flat = torch.cat([t_.reshape(-1) for t_ in grads.values()])
                dist.all_reduce(flat, op=dist.ReduceOp.AVG)

    def step():
        y, grads, dx = compute()
        exchange(grads)
        return y, grads, dx

    def timed(fn, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(k)]
        for i in range(k):
            flush_l2(flush, i)
            evs[i][0].record(stream)
            fn()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # kernels of ours per step (counted on an eager step; graph replays launch the same set)
    l0 = _lib.launch_count()
    step()
    torch.cuda.synchronize()
    per_step_launches = _lib.launch_count() - l0
    run = step
    if not args.no_graph:
        # the whole compute step (pack + fwd + bwd) as one CUDA graph:
        # no host launch gaps between the ~8 kernels
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            compute()
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            _, g_static, _ = compute()
            exchange(g_static)  # the NCCL all-reduce is part of the replayed step

        def run():
            graph.replay()
        for _ in range(args.warmup):
            run()
    torch.cuda.synchronize()
    if _dist(world):
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = timed(run, args.steps)
    launches = per_step_launches * args.steps
    if _dist(world):
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = sum(ms)
    if _dist(world):
        tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / args.steps
    clocks = sampled_clocks(local, clk, run, ms_step, world)
    flops = flops_of(wl)
    value = world * flops / (ms_step * 1e-3) / 1e12

    # ---- per-kernel timing: the library records a CUDA event after each of its
    # launches (qd_profile); captured into a graph of the step and replayed, so
    # the intervals are kernel durations on the launching stream ----
    pk = load_peaks()
    lib = _lib.load()
    pgraph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        compute()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    # the timed step runs the v3 wgrad and the dgrad concurrently on disjoint SM
    # partitions; per-kernel durations are taken with each kernel alone on all SMs
    # (marks on one stream), which is what the roofline of a kernel means
    part_env = os.environ.get("QD_NO_PART")
    os.environ["QD_NO_PART"] = "1"
    os.environ["QD_FOLD_MAIN"] = "1"  # the wgrad fold on the same stream (one chain of marks)
    lib.qd_profile(1)  # marks from here on: [begin, kernel_1, ..., kernel_k] of the captured step
    with torch.cuda.graph(pgraph):
        lib.qd_profile_mark(torch.cuda.current_stream().cuda_stream)
        compute()
    lib.qd_profile(0)
    del os.environ["QD_FOLD_MAIN"]
    if part_env is None:
        del os.environ["QD_NO_PART"]
    else:
        os.environ["QD_NO_PART"] = part_env
    acc = {}
    reps = max(5, args.steps)
    for _ in range(reps):
        flush_l2(flush, 7)
        pgraph.replay()
        torch.cuda.synchronize()
        seen = {}
        for nm, t in _lib.profile_read():
            k = nm
            if nm == "conv2" or nm == "conv_gemm":
                k = nm + ("[fprop]" if seen.get(nm, 0) == 0 else "[dgrad]")
                seen[nm] = seen.get(nm, 0) + 1
            acc.setdefault(k, []).append(t)
    kern = {k: sum(v) / len(v) for k, v in acc.items()}
    third = flops / 3.0  # fprop, dgrad and wgrad each carry one third of the GEMM work
    tensor_k = {k: v for k, v in kern.items()
                if k.split("[")[0] in ("conv2", "conv_gemm", "wgrad2", "wgrad3", "wgrad_v1", "simt_gemm")}
    es = 2 if dts == "bf16" else 4
    m_out = n * ((h + 2 * p - r) // s + 1) * ((w + 2 * p - r) // s + 1)
    kernels = {}
    for k, v in kern.items():
        e = {"ms": v}
        if k in tensor_k:
            e["tflops"] = third / (v * 1e-3) / 1e12
        elif k.startswith("prologue"):
            # reads dy, a, b (3 F channels); writes D: [g b | g a] (2 F) for proposed at
            # stride 1 (the GEMMs read g from dy), [g b | g a | g] (3 F) otherwise; t4 2 F
            wcols = 2 * f if (fam == "t4" or (fam == "proposed" and s == 1)) else 3 * f
            e["gbs"] = (3 * f + wcols) * m_out * es / (v * 1e-3) / 1e9
            e["bytes"] = (3 * f + wcols) * m_out * es
        kernels[k] = e
    dom = max(tensor_k, key=lambda k_: tensor_k[k_]) if tensor_k else max(kern, key=lambda k_: kern[k_])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            ncu = json.load(fh)
        ent = ncu.get("kernels", {}).get(dom.split("[")[0] + ("[" + dom.split("[")[1] if "[" in dom else ""))
        if ent and ent.get("workload") == wl_name:
            traffic = ent["dram_bytes"]
    except Exception:  # noqa: BLE001
        traffic = None
    ach = third / (kern[dom] * 1e-3) / 1e12
    roof = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": pk["bf16"],
            "unit": "TFLOP/s", "frac": ach / pk["bf16"], "traffic": traffic,
            "peak_src": f"{pk['src']} bf16 dense burst ({pk['bf16']}); sustained {pk['bf16_sustained']}",
            "kernels": kernels,
            "algorithmic": "per launch: 1/3 of 9 x 2*M*K*F (one GEMM set); traffic = ncu dram read+write "
                           "of the same kernel (profiles/ncu_summary.json)",
            "timing": "kernel durations from CUDA events on the launching stream, each kernel alone on all "
                      "SMs (QD_NO_PART; the split-K fold then runs as wsum + bwd_finish); the timed step "
                      "overlaps wgrad3 and dgrad on disjoint SM partitions, the partitioned wgrad3 folding "
                      "its partials in-kernel"}
    if kind == "dwconv":
        # depth-wise: r*r MACs per output element -- HBM-bound elementwise-like kernels;
        # algorithmic bytes per launch in units of one (M x C) activation tensor
        unit = m_out * c * es
        per = {"dw_fwd": 4, "prologue": 6, "dw_wgrad": 4, "dw_dgrad": 4}  # x->y,a,b; dy,a,b->D; x,D; D->dx
        for k_, e in kernels.items():
            if k_ in per:
                e["bytes"] = per[k_] * unit
                e["gbs"] = e["bytes"] / (e["ms"] * 1e-3) / 1e9
        dk = max((k_ for k_ in kernels if k_ in per), key=lambda k_: kernels[k_]["ms"])
        roof = {"bound": "hbm", "kernel": dk, "achieved": kernels[dk]["gbs"], "peak": pk["hbm"], "unit": "GB/s",
                "frac": kernels[dk]["gbs"] / pk["hbm"], "traffic": None, "kernels": kernels,
                "peak_src": f"{pk['src']} HBM copy bandwidth",
                "algorithmic": "per launch: the activation tensors the kernel must read and write once "
                               "(dw_fwd x -> y, a, b; prologue dy, a, b -> D; dw_wgrad x, D; dw_dgrad D -> dx)"}
    elif dts != "bf16" and neurons.device_path(spec, x.shape, dt) == 3:
        # fp32 as split bf16 operands: 3 bf16 MMA products per fp32 product, so the ceiling
        # of this path is a third of the bf16 tensor peak (same unit: fp32-equivalent FLOPs)
        roof["peak"] = pk["bf16"] / 3.0
        roof["frac"] = ach / roof["peak"]
        roof["peak_src"] = (f"{pk['src']} bf16 dense burst {pk['bf16']} / 3 (three bf16 products per fp32 "
                            f"product); TF32 for comparison: {TF32_PEAK} (cuBLAS, profiles/r2_tf32_peak.json)")
        roof["note"] = ("fp32 on the tcgen05 kernels: operands split into bf16 hi + lo, products hi*hi + hi*lo "
                        "+ lo*hi accumulated in fp32 (error ~1e-5, tolerance 1e-4)")
    elif dts != "bf16":
        roof["note"] = "fp32 runs on the CUDA-core (FFMA) path; the bf16 tensor peak is the denominator"

    # ---- end to end through the public API with host buffers ----
    x_h = x.detach().cpu().pin_memory()
    g_h = gy.detach().cpu().pin_memory()
    w_h = {k_: v.detach().cpu().pin_memory() for k_, v in params.items()}
    dx_h = (torch.empty(x.shape, dtype=dt) if kind == "fc" else
            torch.empty(x.shape, dtype=dt, memory_format=torch.channels_last)).pin_memory()
    gr_h = {k_: torch.empty(v.shape, dtype=torch.float32).pin_memory() for k_, v in params.items()}

    bufs = [{"x": torch.empty_like(x), "g": torch.empty_like(gy),
             "w": {k_: torch.empty_like(v) for k_, v in params.items()}} for _ in range(2)]

    def h2d_in(b):
        bufs[b]["x"].copy_(x_h, non_blocking=True)
        bufs[b]["g"].copy_(g_h, non_blocking=True)
        for k_, v in w_h.items():
            bufs[b]["w"][k_].copy_(v, non_blocking=True)

    def compute_e2e(b):
        yy, cc = neurons.forward(spec, bufs[b]["w"], bufs[b]["x"], dtype=dt)
        grads, dxx = neurons.symbolic_backward(spec, bufs[b]["w"], cc, bufs[b]["g"])
        exchange(grads)
        return [dxx] + [grads[k_] for k_ in gr_h]

    def d2h_out(outs):
        dx_h.copy_(outs[0], non_blocking=True)
        for k_, v in zip(gr_h, outs[1:]):
            gr_h[k_].copy_(v, non_blocking=True)

    pipelined_e2e(max(10, 2 * args.warmup), h2d_in, compute_e2e, d2h_out)  # warm-up (PCIe link and copy engines at speed)
    e2e_step_ms = pipelined_e2e(args.steps, h2d_in, compute_e2e, d2h_out)
    if _dist(world):
        tt = torch.tensor([e2e_step_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_step_ms = float(tt.item())
    h2d = x_h.numel() * x_h.element_size() + g_h.numel() * g_h.element_size() + sum(
        v.numel() * 4 for v in w_h.values())
    d2h = dx_h.numel() * dx_h.element_size() + sum(v.numel() * 4 for v in gr_h.values())

    # the data-parallel training config the scaling target names (BASELINE.json:
    # QuadraResNet-18 img/s at 1/2/4/8 GPUs), measured in the same run at this N
    nets = {}
    for net in args.nets:
        nets[net] = measure_net(args, net, world, rank, local, dev)

    if _dist(world):
        dist.barrier()
    if rank != 0:
        if _dist(world):
            dist.destroy_process_group()
        return 0

    # ---- CPU baseline on rank 0 at N=1, bounded sample ----
    cpu = None
    if world == 1 and not args.no_cpu:
        batch = cpu_batch_for(wl)
        t_cpu, fl = cpu_sample(wl, batch, 2)
        cpu = {"value": fl / t_cpu / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count(),
               "kind": "port",
               "sample": f"{wl_name} at batch {batch} of {n}, fp64 numpy reference algorithm "
                         f"(im2col+GEMM+col2im), best of 2, {t_cpu:.2f} s"}
    out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": dts, "data": "synthetic (seeded N(0,1) x and dy, Kaiming-uniform W, b=0)",
           "config": config_of(wl, wl_name, world), "cuda_graph": not args.no_graph,
           "roofline": roof, "cpu_baseline": cpu,
           "e2e": {"value": world * flops / (e2e_step_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                   "ms_per_step": e2e_step_ms, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h,
                   "note": "public API (neurons.forward / symbolic_backward); every step copies its x, dy and fp32 "
                           "weights from pinned host memory and dx and the fp32 gradients back; double-buffered "
                           "inputs on a copy stream overlap step i+1's H2D with step i's compute and D2H; no L2 "
                           "flush inside the loop (inputs arrive over PCIe every step, the step's own traffic "
                           "exceeds L2)"},
           "gpu_launches": launches, "launches_per_step": launches / args.steps,
           "clocks": clocks, "nets": nets,
           "path": {0: "cuda-core", 1: "tcgen05", 2: "depth-wise", 3: "tcgen05 fp32 (split bf16 x3)"}[
               neurons.device_path(spec, x.shape, dt)]}
    print(json.dumps(out), flush=True)
    if _dist(world):
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# network training step (BASELINE configs 3 and 4): img/s
# ---------------------------------------------------------------------------
NETS = {
    # name: (builder, per-GPU batch, image HW, classes)
    "qvgg16": ("QuadraVGG16", 256, 32, 10),
    "qresnet18": ("QuadraResNet18", 128, 224, 1000),
}


def net_quad_layers(name):
    """(spec, input CHW) of every quadratic conv in the net, for FLOP counting and
    the CPU baseline (built on the meta device: shapes only)."""
    import torch
    from paper_2204_01701_b200 import qnets
    from paper_2204_01701_b200.nn import QuadConv2d
    builder, batch, hw, classes = NETS[name]
    shapes = []
    hooks = []
    with torch.device("meta"):
        model = getattr(qnets, builder)(num_classes=classes)
    inner = set()
    from paper_2204_01701_b200.im2col import Im2colConv2d
    for m in model.modules():
        if isinstance(m, Im2colConv2d) and m.conv_spec.family != "first_order":
            # algorithmic work of the conv itself (real input channels, not the K padding)
            hooks.append(m.register_forward_pre_hook(
                lambda mod, inp: shapes.append((mod.conv_spec, tuple(inp[0].shape[1:])))))
    from paper_2204_01701_b200.bn import QuadConvBN
    for m in model.modules():
        if isinstance(m, QuadConvBN):  # fused conv -> BN (-> ReLU) node: its layer never runs forward()
            # (the first-order 1x1 shortcuts are not quadratic layers)
            hooks.append(m.register_forward_pre_hook(
                lambda mod, inp: shapes.append((mod.layer.spec, tuple(inp[0].shape[1:])))
                if mod.layer.spec.family != "first_order" else None))
        elif isinstance(m, QuadConv2d) and id(m) not in inner:
            hooks.append(m.register_forward_pre_hook(
                lambda mod, inp: shapes.append((mod.spec, tuple(inp[0].shape[1:])))))
    # trace shapes with a meta-device forward that bypasses the kernels
    import paper_2204_01701_b200.bn as qbn
    import paper_2204_01701_b200.nn as qnn
    orig, orig_bn = qnn.QuadFunction.apply, qbn._QuadBNFunction.apply

    def fake(spec, dtype, x, *ts):
        oh = (x.shape[2] + 2 * spec.pad - spec.kernel) // spec.stride + 1
        ow = (x.shape[3] + 2 * spec.pad - spec.kernel) // spec.stride + 1
        return torch.empty(x.shape[0], spec.out_dim, oh, ow, device=x.device)

    def fake_bn(spec, dtype, relu, bn, x, *ts):
        return fake(spec, dtype, x)
    qnn.QuadFunction.apply = fake
    qbn._QuadBNFunction.apply = fake_bn
    try:
        with torch.device("meta"):
            model(torch.empty(1, 3, hw, hw))
    finally:
        qnn.QuadFunction.apply = orig
        qbn._QuadBNFunction.apply = orig_bn
        for h in hooks:
            h.remove()
    return shapes


def net_flops(name, batch):
    from paper_2204_01701_b200.spec import gemm_flops
    return sum(gemm_flops(sp, batch, c_hw[1], c_hw[2]) for sp, c_hw in net_quad_layers(name))


def net_cpu_baseline(name):
    """Reference algorithm (oracle port) fwd+bwd of every quadratic layer at batch 1,
    summed: seconds per image (linear in N)."""
    from oracle import quadra_oracle as Q
    tot = 0.0
    for sp, (c, h, w) in net_quad_layers(name):
        fam = sp.family
        x, P, g = Q.synthetic_layer(fam, "conv", 1, c, sp.out_dim, h, w, sp.kernel, sp.stride, sp.pad, seed=0)
        geo = Q.Geometry("conv", sp.kernel, sp.stride, sp.pad)
        t0 = time.perf_counter()
        y, a, b = Q.forward(fam, geo, P, x)
        Q.symbolic_backward(fam, geo, P, x, a, b, g)
        tot += time.perf_counter() - t0
    return tot


def run_net(args, name):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if _dist(world):
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    out = measure_net(args, name, world, rank, local, dev)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if _dist(world):
        dist.destroy_process_group()
    return 0


def measure_net(args, name, world, rank, local, dev):
    """One QuadraNet training-step measurement on every rank (the process group,
    if any, is already up); returns rank 0's JSON object (None on other ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2204_01701_b200 import _lib, qnets
    from paper_2204_01701_b200.dp import BucketedAllReduce, broadcast_module, sgd
    from paper_2204_01701_b200.optim import QuadSGD

    builder, batch, hw, classes = NETS[name]
    batch = args.batch or batch
    # the first-order convs (ResNet stem, 1x1 shortcuts) run on cuDNN: let it time
    # its algorithms for these fixed shapes once instead of taking its heuristic pick
    torch.backends.cudnn.benchmark = os.environ.get("QD_CUDNN_BENCH", "1") == "1"
    torch.manual_seed(1234)
    model = getattr(qnets, builder)(num_classes=classes).to(dev).to(memory_format=torch.channels_last)
    broadcast_module(model)  # every replica starts from rank 0's weights and BN buffers
    # fused SGD + weight pack for the quadratic layers;
    # --torch-sgd for torch.optim.SGD everywhere (the forward then packs itself)
    for p_ in model.parameters():  # activations are channels_last; parameters keep the standard layout
        p_.data = p_.data.contiguous()
    opt = sgd(model.parameters(), lr=0.01) if args.torch_sgd else QuadSGD(model, lr=0.01)
    red = BucketedAllReduce(model.parameters(), bucket_mb=25.0)
    gen = torch.Generator(device=dev).manual_seed(rank)
    x = torch.randn(batch, 3, hw, hw, device=dev, generator=gen).to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    y = torch.randint(0, classes, (batch,), device=dev, generator=gen)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def eager_step(xb=x, yb=y):
        red.reset()
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):
            loss = torch.nn.functional.cross_entropy(model(xb), yb)
        loss.backward()
        red.finish()
        opt.step()
        return loss

    # the whole training step (forward, loss, backward with the bucketed all-reduce
    # hooks, fused SGD + pack) captured once as a CUDA graph and replayed: the
    # eager step is host-bound (hundreds of launches from Python). Inputs are
    # static buffers the e2e leg refills from pinned host memory every step.
    graph = None
    launches_graph = None
    if not args.no_graph:
        from paper_2204_01701_b200.graphstep import GraphedStep
        ok = 1
        try:
            gs = GraphedStep(eager_step, x, y, warmup=3, counter=_lib.launch_count)
            launches_graph = gs.captured_launches
        except Exception as e:  # noqa: BLE001 - reported, then the eager step is timed
            print(f"[bench] CUDA-graph capture failed ({type(e).__name__}: {e}); timing the eager step",
                  file=sys.stderr)
            ok = 0
        if _dist(world):  # every rank must take the same path
            t = torch.tensor([ok], device=dev, dtype=torch.int32)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            ok = int(t.item())
        if ok:
            graph = gs

    def step(xb=None, yb=None):
        if graph is None:
            return eager_step(x if xb is None else xb, y if yb is None else yb)
        return graph(xb, yb)

    def timed(fn, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        for i in range(k):
            flush_l2(flush, i)
            evs[i][0].record(stream)
            fn()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in evs]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    step()
    torch.cuda.synchronize()
    per_step = launches_graph if graph is not None else _lib.launch_count() - l0
    if _dist(world):
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = timed(step, args.steps)
    tot = sum(ms)
    if _dist(world):
        tt = torch.tensor([tot], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tot = float(tt.item())
    ms_step = tot / args.steps
    clocks = sampled_clocks(local, clk, step, ms_step, world, seconds=1.0)
    value = world * batch / (ms_step * 1e-3)
    qflops = net_flops(name, batch)
    pk = load_peaks()
    ach = qflops / (ms_step * 1e-3) / 1e12

    # e2e: batch from pinned host memory each step, loss read back
    x_h = x.detach().cpu().pin_memory()
    y_h = y.detach().cpu().pin_memory()
    loss_h = torch.empty((), dtype=torch.float32).pin_memory()

    stage = [(torch.empty_like(x), torch.empty_like(y)) for _ in range(2)]

    def h2d_in(b):
        stage[b][0].copy_(x_h, non_blocking=True)
        stage[b][1].copy_(y_h, non_blocking=True)

    def compute_e2e(b):
        return [step(stage[b][0], stage[b][1]).detach()]

    def d2h_out(outs):
        loss_h.copy_(outs[0].float(), non_blocking=True)

    pipelined_e2e(max(10, 2 * args.warmup), h2d_in, compute_e2e, d2h_out)  # warm-up (PCIe link and copy engines at speed)
    e_step = pipelined_e2e(args.steps, h2d_in, compute_e2e, d2h_out)
    if _dist(world):
        tt = torch.tensor([e_step], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e_step = float(tt.item())
    if _dist(world):
        dist.barrier()
    red.remove()
    if rank != 0:
        return None
    cpu = None
    if world == 1 and not args.no_cpu:
        sec = net_cpu_baseline(name)
        cpu = {"value": 1.0 / sec, "unit": "img/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"reference algorithm (fp64 im2col+GEMM+col2im) fwd+bwd of the {len(net_quad_layers(name))} "
                         f"quadratic layers of {name} at batch 1, summed ({sec:.2f} s/img; linear in batch, "
                         "BASELINE.md §4); first-order layers not counted"}
    out = {"metric": f"{name}_train_img_per_s", "value": value, "unit": "img/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic (seeded N(0,1) images, uniform labels)",
           "config": {"workload": f"{name}: full training step (fwd, CE loss, bwd, bucketed all-reduce, "
                                  f"SGD m=0.9 wd=5e-4)", "global_batch": batch * world, "per_gpu_batch": batch,
                      "image": [3, hw, hw], "classes": classes, "parallelism": f"dp{world}",
                      "l2": L2_NOTE, "cuda_graph": graph is not None,
                      "params": qnets.count_params(model), "quad_gemm_flops_per_gpu_step": qflops},
           "roofline": {"bound": "tensor", "kernel": "all quadratic-layer GEMM work of the step",
                        "achieved": ach, "peak": pk["bf16"], "unit": "TFLOP/s", "frac": ach / pk["bf16"],
                        "traffic": None,
                        "note": "whole-step figure: quadratic GEMM FLOPs / step time (first-order layers, BN, "
                                "optimizer and all-reduce included in the time)"},
           "cpu_baseline": cpu,
           "e2e": {"value": world * batch / (e_step * 1e-3), "unit": "img/s", "ms_per_step": e_step,
                   "h2d_bytes_per_step": x_h.numel() * x_h.element_size() + y_h.numel() * y_h.element_size(),
                   "d2h_bytes_per_step": 4,
                   "note": "every step copies its image batch and labels from pinned host memory (double-buffered "
                           "on a copy stream, overlapping the previous step's compute) into the graph's input "
                           "buffers and reads the loss back"},
           "gpu_launches": per_step * args.steps, "launches_per_step": per_step, "clocks": clocks}
    return out


def run_net_reference(args, name):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    builder, batch, hw, classes = NETS[name]
    times = [net_cpu_baseline(name) for _ in range(max(1, args.steps))]
    sec = sum(times) / len(times)
    value = 1.0 / sec
    # ms_per_step: the MEASURED time of one step of the bounded sample (every quadratic
    # layer at batch 1, `step_batch`); value is its rate (linear in the batch)
    out = {"metric": f"{name}_train_img_per_s", "value": value, "unit": "img/s", "impl": "reference",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
           "step_batch": 1,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{name}: quadratic layers fwd+bwd, batch 1 sample scaled", "per_gpu_batch": batch},
           "cpu_baseline": {"value": value, "unit": "img/s", "cores": os.cpu_count(), "kind": "port",
                            "sample": "quadratic layers at batch 1 (reference algorithm)"},
           "e2e": {"value": value, "unit": "img/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS) + sorted(NETS))
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch for the net workloads")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--torch-sgd", action="store_true", help="nets: torch.optim.SGD instead of the fused SGD+pack")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly (no CUDA graph)")
    ap.add_argument("--nets", default=None,
                    help="layer workloads: comma list of net training steps measured in the same run and "
                         "reported under 'nets' (default: qresnet18 for c2, none otherwise; '' = none)")
    args = ap.parse_args()
    if args.nets is None:
        args.nets = "qresnet18" if args.workload == "c2" else ""
    args.nets = [n for n in args.nets.split(",") if n]
    for n in args.nets:
        if n not in NETS:
            ap.error(f"--nets: unknown net {n!r}")
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.workload in NETS:
        if args.impl == "reference":
            return run_net_reference(args, args.workload)
        return run_net(args, args.workload)
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, wl, args.workload)
    return run_ours(args, wl, args.workload)


if __name__ == "__main__":
    sys.exit(main())
