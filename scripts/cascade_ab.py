"""Fused cascade vs per-layer path (Cascade._fused = None) for a few stacks:
forward + backward per step, CUDA events.  One JSON line per stack.

  python scripts/cascade_ab.py
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import AcdcLayer, Cascade, PermutationLayer, ReluLayer  # noqa: E402


def stack(n, depth, relu_perm, dev, rng):
    layers = []
    for i in range(depth):
        L = AcdcLayer(n, device=dev)
        L.a.normal_(1.0, 0.061)
        L.d.normal_(1.0, 0.061)
        layers.append(L)
        if relu_perm and i < depth - 1:
            layers += [ReluLayer(n, device=dev), PermutationLayer(n, perm=rng.permutation(n), device=dev)]
    return Cascade(layers)


def timeit(fn, steps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def graphed(step):
    step()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        step()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            step()
    torch.cuda.synchronize()
    return g.replay


def main():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    for n, depth, rows, rp in ((4096, 32, 4096, False), (4096, 12, 4096, True), (2048, 12, 8192, True),
                               (2048, 32, 8192, False), (1024, 12, 8192, True)):
        casc = stack(n, depth, rp, dev, rng)
        x = torch.randn(rows, n, device=dev)
        dy = torch.randn(rows, n, device=dev)

        def step():
            casc.forward(x)
            casc.backward(dy)

        fused = casc._fused
        ms_f = timeit(step)
        ms_fg = timeit(graphed(step))
        casc._fused = None
        ms_u = timeit(step)
        ms_ug = timeit(graphed(step))
        casc._fused = fused
        print(json.dumps({"n": n, "depth": depth, "rows": rows, "relu_perm": rp, "fused_ms": ms_f,
                          "per_layer_ms": ms_u, "fused_graph_ms": ms_fg, "per_layer_graph_ms": ms_ug,
                          "per_layer_over_fused_graph": ms_ug / ms_fg}), flush=True)
        del casc
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
