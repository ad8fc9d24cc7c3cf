"""Probe: where the time of the tiny C1 step (N=256, 128 rows) goes.

CUDA-graph replays of the forward alone, the backward (+ reduction) alone and
the whole step; one JSON line.

  python scripts/c1_probe.py [n] [rows]
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import functional as F  # noqa: E402


def graph_us(fn, reps=2000):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    dev = torch.device("cuda", 0)
    F.prepare(n, dev)
    x = torch.randn(rows, n, device=dev)
    dy = torch.randn(rows, n, device=dev)
    a, d, b = (torch.randn(n, device=dev) for _ in range(3))
    g = torch.zeros(3, n, device=dev)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    hc = F.new_h2cache(rows, n, dev) if F.h2cache_supported(n) else None
    fwd = lambda: F.acdc_forward(x, a, d, b, out=y, h2cache=hc)  # noqa: E731
    bwd = lambda: F.acdc_backward(x, dy, a, d, g[0], g[1], g[2], accumulate=False, out=dx, h2cache=hc)  # noqa: E731
    empty = torch.empty(1, device=dev)
    res = {"n": n, "rows": rows, "h2cache": hc is not None,
           "fwd_us": graph_us(fwd), "bwd_us": graph_us(bwd),
           "step_us": graph_us(lambda: (fwd(), bwd())),
           "noop_kernel_us": graph_us(lambda: empty.add_(1.0)),
           "bwd_launches": F._lib.load().acdc_bwd_launch_count(rows, n, 1 if hc is not None else 0)}
    if rows <= F.step_max_rows(n):  # the fused one-launch step (acdc_step_f32)
        res["fused_step_us"] = graph_us(lambda: F.acdc_step(x, dy, a, d, b, g[0], g[1], g[2], accumulate=False,
                                                           out_y=y, out_dx=dx))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
