"""Secondary benchmarks for the other BASELINE.json configs (one JSON line each).

    python bench_configs.py [--only c1,sweep,c3,c4,c5] [--steps K]

C1    single layer N=256, batch 128, fwd+bwd (launch-bound: CUDA-graph replay)
      next to the reference CPU path (oracle/_ref, all host threads)
sweep single layer N=128..32768, batch 16384: rows/s and % of the 20N HBM
      roofline, next to a cuBLAS dense linear of the same N (fp32 and TF32)
C3    12-block ACDC+ReLU+Perm cascade, N=1024, batch 8192: fused vs per-layer
C4    deep SELL training step: 32 ACDC layers at N=4096 (fused cascade), MSE
      loss gradient and momentum SGD on the diagonals, batch 4096 per GPU
C5    complex AFDF N=8192, 8192 rows per GPU (65536 over 8 GPUs)
Timing: CUDA events around K steps after warm-up; inputs larger than L2 or
already L2-resident as stated per line.
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


def c1(args, dev):
    n, B = 256, 128
    step, mode = layer_step(n, B, dev)
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
    ms_graph = timeit(graph.replay, args.steps * 10)
    ms_eager = timeit(step, args.steps * 10)
    from bench import cpu_threads, reference_cpu

    thr = cpu_threads()
    rps_cpu, kind, sample, _, used = reference_cpu(n, min(thr, 8), B, seconds=3.0, warmup=1)
    rps = B / (ms_graph / 1e3)
    return {"config": "C1 single ACDC layer N=256 batch 128 fwd+bwd", "mode": mode, "us_per_step_graph": ms_graph * 1e3,
            "us_per_step_eager": ms_eager * 1e3, "rows_per_s": rps,
            "cpu_reference": {"rows_per_s": rps_cpu, "kind": kind, "threads": used, "sample": sample},
            "speedup_vs_cpu": rps / rps_cpu}


def sweep(args, dev):
    out = []
    hbm = peak_hbm()
    for lg in range(7, 16):
        n = 1 << lg
        B = 16384
        step, mode = layer_step(n, B, dev)
        ms = timeit(step, args.steps)
        rps = B / (ms / 1e3)
        row = {"config": "sweep single ACDC layer fwd+bwd batch 16384", "n": n, "mode": mode, "ms_per_step": ms,
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

    ms_f = timeit(step, args.steps)
    fused = casc._fused
    casc._fused = None
    ms_u = timeit(step, max(3, args.steps // 4))
    casc._fused = fused
    # bytes: x, y, dy, dx (16N) + checkpoints x_l (K-1) and h2_l (K) written once, read once
    bytes_row = 16 * n + 2 * 4 * n * ((depth - 1) + depth)
    return {"config": "C3 12-block ACDC+ReLU+Perm cascade N=1024 batch 8192", "fused_ms": ms_f, "unfused_ms": ms_u,
            "fused_rows_per_s": B / (ms_f / 1e3), "unfused_rows_per_s": B / (ms_u / 1e3),
            "fused_speedup": ms_u / ms_f, "fused_bytes_per_row": bytes_row,
            "fused_hbm_frac": B / (ms_f / 1e3) * bytes_row / (peak_hbm() * 1e9)}


def c4(args, dev):
    """Deep SELL step: forward, MSE loss gradient, backward, momentum SGD (training.py:72-84)."""
    n, depth, B = 4096, 32, 4096
    rng = np.random.default_rng(1)
    casc, layers = _cascade(n, depth, False, dev, rng)
    x = torch.randn(B, n, device=dev)
    target = torch.randn(B, n, device=dev)
    from paper_1511_05946_b200.training import Sgd, SgdConfig

    opt = Sgd(casc.params(), SgdConfig(learning_rate=1e-3, momentum=0.9))  # training.py:58-84

    def step():
        y = casc.forward(x)
        gy = (2.0 / y.numel()) * (y - target)  # mse_loss gradient (training.py:176-183)
        casc.backward(gy)
        opt.step()  # momentum SGD, zeroes the grads

    def step_fused():  # the SGD update inside each block's gradient reduction (acdc_bwd_sgd_f32)
        y = casc.forward(x)
        gy = (2.0 / y.numel()) * (y - target)
        opt.backward_step(casc, gy)

    ms = timeit(step, max(3, args.steps // 10))
    ms_f = timeit(step_fused, max(3, args.steps // 10))
    return {"config": "C4 deep SELL 32 ACDC layers N=4096 train step (1 GPU of the DP job)", "fused": casc.fused,
            "batch_per_gpu": B, "ms_per_step": ms, "rows_per_s": B / (ms / 1e3),
            "layer_rows_per_s": B * depth / (ms / 1e3),
            "fused_sgd": {"ms_per_step": ms_f, "rows_per_s": B / (ms_f / 1e3)}}


def c5(args, dev):
    n, B = 8192, 8192
    x = torch.randn(B, n, dtype=torch.complex64, device=dev)
    dy = torch.randn(B, n, dtype=torch.complex64, device=dev)
    a = (1 + 0.1 * torch.randn(n, device=dev)) + 0.1j * torch.randn(n, device=dev)
    d = (1 + 0.1 * torch.randn(n, device=dev)) + 0.1j * torch.randn(n, device=dev)
    ga = torch.zeros(n, dtype=torch.complex64, device=dev)
    gd = torch.zeros_like(ga)
    y, dx = torch.empty_like(x), torch.empty_like(x)

    def step():
        F.afdf_forward(x, a, d, out=y)
        F.afdf_backward(x, dy, a.to(torch.complex64), d.to(torch.complex64), ga, gd, accumulate=False, out=dx)

    ms = timeit(step, args.steps)
    rps = B / (ms / 1e3)
    return {"config": "C5 AFDF N=8192 complex64, 8192 rows per GPU (65536 over 8)", "ms_per_step": ms,
            "rows_per_s_per_gpu": rps, "bytes_per_row": 40 * n,
            "hbm_roofline_frac": rps * 40 * n / (peak_hbm() * 1e9)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,sweep,c3,c4,c5")
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    for name in args.only.split(","):
        res = globals()[name](args, dev)
        for r in (res if isinstance(res, list) else [res]):
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
