"""Secondary benchmarks for the other BASELINE.json configs (one JSON line each).

    python bench_configs.py [--only c1,sweep,c3,c4,c5] [--steps K]

C1    single layer N=256, batch 128, fwd+bwd (launch-bound: CUDA-graph replay)
      next to the reference CPU path (oracle/_ref, all host threads)
sweep single layer N=128..32768, batch 16384: rows/s and % of the 20N HBM
      roofline, next to a cuBLAS dense linear of the same N (fp32 and TF32)
C3    12-block ACDC+ReLU+Perm cascade, N=1024, batch 8192: fused vs per-layer
C4    deep SELL training step: 32 ACDC layers at N=4096 (fused cascade), MSE
      loss gradient and momentum SGD on the diagonals, batch 4096 per GPU,
      data-parallel over the ranks (bucketed all-reduce overlapping the backward)
C5    complex AFDF N=8192, 65536 rows in total sharded over the ranks
Timing: CUDA events around K steps after warm-up, max over ranks; inputs
larger than L2 or already L2-resident as stated per line.

    python bench_configs.py --only c4,c5 --gpus 8     (re-launches under torchrun)
C4 / C5 run one process per GPU (NCCL); the other configs run on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1511_05946_b200 import functional as F  # noqa: E402


def peak_hbm():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def timeit(fn, steps, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def layer_step(n, B, dev, mode="auto"):
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    x = torch.randn(B, n, device=dev, generator=g)
    dy = torch.randn(B, n, device=dev, generator=g)
    a = 1 + 0.1 * torch.randn(n, device=dev, generator=g)
    d = 1 + 0.1 * torch.randn(n, device=dev, generator=g)
    b = 0.1 * torch.randn(n, device=dev, generator=g)
    gr = torch.zeros(3, n, device=dev)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    F.prepare(n, dev)
    cache = F.new_h2cache(B, n, dev) if (mode != "recompute" and F.h2cache_supported(n)) else None

    def step():
        F.acdc_forward(x, a, d, b, out=y, h2cache=cache)
        F.acdc_backward(x, dy, a, d, gr[0], gr[1], gr[2], accumulate=False, out=dx, h2cache=cache)

    return step, ("h2cache" if cache is not None else "recompute")


def dense_step(n, B, dev, tf32):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    w = torch.randn(n, n, device=dev) / math.sqrt(n)
    x = torch.randn(B, n, device=dev)
    gy = torch.randn(B, n, device=dev)

    def step():
        x @ w
        gy @ w.t()
        x.t() @ gy

    return step


def fused_step(n, B, dev):
    """The fused small-batch step (functional.acdc_step: forward + backward +
    gradient reduction in ONE launch for a dy known up front, as here)."""
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    x = torch.randn(B, n, device=dev, generator=g)
    dy = torch.randn(B, n, device=dev, generator=g)
    a = 1 + 0.1 * torch.randn(n, device=dev, generator=g)
    d = 1 + 0.1 * torch.randn(n, device=dev, generator=g)
    b = 0.1 * torch.randn(n, device=dev, generator=g)
    gr = torch.zeros(3, n, device=dev)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    F.prepare(n, dev)
    assert B <= F.step_max_rows(n)
    return lambda: F.acdc_step(x, dy, a, d, b, gr[0], gr[1], gr[2], accumulate=False, out_y=y, out_dx=dx)


def graph_of(step):
    step()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        step()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            step()
    torch.cuda.synchronize()
    return graph


def c1(args, dev):
    n, B = 256, 128
    step, mode = layer_step(n, B, dev)
    graph = graph_of(step)
    ms_graph_sep = timeit(graph.replay, args.steps * 10)
    ms_eager_sep = timeit(step, args.steps * 10)
    fstep = fused_step(n, B, dev)
    fgraph = graph_of(fstep)
    ms_graph = timeit(fgraph.replay, args.steps * 10)
    ms_eager = timeit(fstep, args.steps * 10)
    from bench import cpu_threads, reference_cpu

    thr = cpu_threads()
    rps_cpu, kind, sample, _, used = reference_cpu(n, min(thr, 8), B, seconds=3.0, warmup=1)
    rps = B / (ms_graph / 1e3)
    return {"config": "C1 single ACDC layer N=256 batch 128 fwd+bwd", "mode": "fused step (acdc_step_f32, 1 launch)",
            "us_per_step_graph": ms_graph * 1e3, "us_per_step_eager": ms_eager * 1e3, "rows_per_s": rps,
            "separate_calls": {"mode": mode, "launches": 3, "us_per_step_graph": ms_graph_sep * 1e3,
                               "us_per_step_eager": ms_eager_sep * 1e3},
            "cpu_reference": {"rows_per_s": rps_cpu, "kind": kind, "threads": used, "sample": sample},
            "speedup_vs_cpu": rps / rps_cpu}


def graphed(step):
    """The step captured once in a CUDA graph (the kernels' programmatic
    dependent launches are kept); replaying it removes the Python / ctypes
    launch overhead, which exceeds the GPU time at small N."""
    step()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        step()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            step()
    torch.cuda.synchronize()
    return graph.replay


def sweep(args, dev):
    out = []
    hbm = peak_hbm()
    for lg in range(7, 16):
        n = 1 << lg
        B = 16384
        step, mode = layer_step(n, B, dev)
        ms_eager = timeit(step, args.steps)
        ms = timeit(graphed(step), args.steps)
        rps = B / (ms / 1e3)
        row = {"config": "sweep single ACDC layer fwd+bwd batch 16384 (CUDA-graph replay)", "n": n, "mode": mode,
               "ms_per_step": ms, "ms_per_step_eager": ms_eager,
               "rows_per_s": rps, "hbm_roofline_frac_20N": rps * 20 * n / (hbm * 1e9)}
        if n <= 8192:
            for tf32 in (False, True):
                dms = timeit(dense_step(n, B, dev, tf32), max(2, args.steps // 20), warmup=1)
                row["dense_" + ("tf32" if tf32 else "fp32")] = {"ms_per_step": dms, "rows_per_s": B / (dms / 1e3),
                                                                 "acdc_speedup": dms / ms}
            torch.backends.cuda.matmul.allow_tf32 = False
        del step
        torch.cuda.empty_cache()
        out.append(row)
    return out


def _cascade(n, depth, relu_perm, dev, rng):
    from paper_1511_05946_b200 import AcdcLayer, Cascade, PermutationLayer, ReluLayer

    layers = []
    for i in range(depth):
        L = AcdcLayer(n, device=dev)
        L.a.normal_(1.0, 0.061)  # PAPER.md:340 init N(1, 0.061)
        L.d.normal_(1.0, 0.061)
        layers.append(L)
        if relu_perm and i < depth - 1:
            layers += [ReluLayer(n, device=dev), PermutationLayer(n, perm=rng.permutation(n), device=dev)]
    return Cascade(layers), layers


def c3(args, dev):
    n, depth, B = 1024, 12, 8192
    rng = np.random.default_rng(0)
    casc, layers = _cascade(n, depth, True, dev, rng)
    x = torch.randn(B, n, device=dev)
    dy = torch.randn(B, n, device=dev)

    def step():
        casc.forward(x)
        casc.backward(dy)

    ms_f_eager = timeit(step, args.steps)
    ms_f = timeit(graphed(step), args.steps)  # the same step replayed from a CUDA graph
    fused = casc._fused
    casc._fused = None
    ms_u = timeit(step, max(3, args.steps // 4))
    casc._fused = fused
    # bytes: x, y, dy, dx (16N) + checkpoints x_l (K-1) and h2_l (K) written once, read once
    bytes_row = 16 * n + 2 * 4 * n * ((depth - 1) + depth)
    return {"config": "C3 12-block ACDC+ReLU+Perm cascade N=1024 batch 8192 (CUDA-graph replay)", "fused_ms": ms_f,
            "fused_ms_eager": ms_f_eager, "unfused_ms": ms_u,
            "fused_rows_per_s": B / (ms_f / 1e3), "unfused_rows_per_s": B / (ms_u / 1e3),
            "fused_speedup": ms_u / ms_f, "fused_bytes_per_row": bytes_row,
            "fused_hbm_frac": B / (ms_f / 1e3) * bytes_row / (peak_hbm() * 1e9)}


def _dist():
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    return world, rank


def timeit_dist(fn, steps, warmup=3):
    """CUDA-event time per step, barrier on both sides, max over ranks."""
    import torch.distributed as dist

    from bench import barrier, max_over_ranks

    world, _ = _dist()
    for _ in range(warmup):
        fn()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    barrier(world)
    return max_over_ranks(e0.elapsed_time(e1), world) / steps


def c4(args, dev):
    """Deep SELL step: forward, MSE loss gradient, backward, momentum SGD
    (training.py:72-84, 210-249), batch-sharded: B rows per rank, parameters
    replicated, gradients summed by DataParallel (one bucketed all-reduce whose
    buckets overlap the backward of the earlier blocks)."""
    from paper_1511_05946_b200.parallel import DataParallel
    from paper_1511_05946_b200.training import Sgd, SgdConfig

    world, rank = _dist()
    n, depth, B = 4096, 32, 4096
    rng = np.random.default_rng(1)  # same parameters on every rank
    casc, layers = _cascade(n, depth, False, dev, rng)
    torch.manual_seed(1)
    for l in layers:  # replicated init (normal_ above used the global generator)
        l.a.normal_(1.0, 0.061)
        l.d.normal_(1.0, 0.061)
    g = torch.Generator(device=dev)
    g.manual_seed(100 + rank)
    x = torch.randn(B, n, device=dev, generator=g)
    target = torch.randn(B, n, device=dev, generator=g)
    dp = DataParallel(casc, bucket_bytes=(args.bucket_kib << 10) if world > 1 else None)
    opt = Sgd(casc.params(), SgdConfig(learning_rate=1e-3, momentum=0.9))  # training.py:58-84
    scale = 2.0 / (B * world * n)  # mse over the global batch (training.py:176-183)

    def step():
        y = dp.forward(x)
        gy = scale * (y - target)
        dp.backward(gy)
        dp.allreduce_grads()
        opt.step()  # momentum SGD on the summed grads, zeroes them

    def step_fused():  # 1 rank only: the SGD update inside each block's gradient reduction
        y = casc.forward(x)
        gy = scale * (y - target)
        opt.backward_step(casc, gy)

    ms = timeit_dist(step, max(3, args.steps // 10))
    res = {"config": f"C4 deep SELL 32 ACDC layers N=4096 train step, {world} GPU(s) data-parallel",
           "n_gpus": world, "fused": casc.fused, "batch_per_gpu": B, "global_batch": B * world, "ms_per_step": ms,
           "rows_per_s": B * world / (ms / 1e3), "layer_rows_per_s": B * world * depth / (ms / 1e3),
           "allreduce": (f"bucketed {args.bucket_kib} KiB, overlapping the backward" if world > 1 else "none"),
           "scaling": "weak"}
    if world == 1:
        ms_f = timeit(step_fused, max(3, args.steps // 10))
        res["fused_sgd"] = {"ms_per_step": ms_f, "rows_per_s": B / (ms_f / 1e3)}
    return res


def c5(args, dev):
    """Complex AFDF N=8192, 65536 rows in total, sharded over the ranks
    (AfdfLayer under DataParallel, layers.py:159-215)."""
    from paper_1511_05946_b200 import AfdfLayer
    from paper_1511_05946_b200.parallel import DataParallel, shard_rows

    world, rank = _dist()
    n, total = 8192, args.c5_rows
    lo, hi = shard_rows(total, world, rank)
    B = hi - lo
    g = torch.Generator(device=dev)
    g.manual_seed(200 + rank)
    x = torch.randn(B, n, dtype=torch.complex64, device=dev, generator=g)
    dy = torch.randn(B, n, dtype=torch.complex64, device=dev, generator=g)
    layer = AfdfLayer(n, device=dev)
    g.manual_seed(7)
    layer.a.copy_((1 + 0.1 * torch.randn(n, device=dev, generator=g)) + 0.1j * torch.randn(n, device=dev, generator=g))
    layer.d.copy_((1 + 0.1 * torch.randn(n, device=dev, generator=g)) + 0.1j * torch.randn(n, device=dev, generator=g))
    dp = DataParallel(layer)

    def step():
        dp.zero_grads()
        dp.forward(x)
        dp.backward(dy)
        dp.allreduce_grads()

    ms = timeit_dist(step, args.steps)
    if world == 1:  # replay of the captured step (eager above: the multi-rank path)
        ms_eager = ms
        ms = timeit(graphed(step), args.steps)
    rps = total / (ms / 1e3)
    return {"config": f"C5 AFDF N=8192 complex64, {total} rows over {world} GPU(s)", "n_gpus": world,
            "timing": "CUDA-graph replay" if world == 1 else "eager",
            **({"ms_per_step_eager": ms_eager} if world == 1 else {}),
            "rows_per_gpu": B, "ms_per_step": ms, "rows_per_s": rps, "rows_per_s_per_gpu": rps / world,
            "bytes_per_row": 40 * n, "hbm_roofline_frac_per_gpu": rps / world * 40 * n / (peak_hbm() * 1e9),
            "scaling": "strong"}


MULTI_GPU = ("c4", "c5")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,sweep,c3,c4,c5")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--bucket-kib", type=int, default=384, help="C4 all-reduce bucket size (8 layers at N=4096)")
    ap.add_argument("--c5-rows", type=int, default=65536)
    args = ap.parse_args()
    from bench import dist_setup, maybe_spawn

    maybe_spawn(args.gpus, __file__)
    world, rank, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local)
    for name in args.only.split(","):
        if world > 1 and name not in MULTI_GPU:
            continue  # single-GPU configs
        res = globals()[name](args, dev)
        if rank == 0:
            for r in (res if isinstance(res, list) else [res]):
                print(json.dumps(r), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
