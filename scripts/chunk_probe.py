"""Probe: a fwd+bwd step over B rows run as L2-resident row chunks.

For chunk size m the step runs, per chunk k, the h2-cache forward on rows
[k*m, (k+1)*m) and then its backward (gradients accumulated).  The chunk's x
and h2 cache (2 * 16 KB per row at N=4096) are still in L2 when the backward
reads them.  Every variant is captured in a CUDA graph and replayed; prints
one JSON line per chunk size.

  python scripts/chunk_probe.py [n] [rows] [chunk ...]
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import functional as F  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    chunks = [int(v) for v in sys.argv[3:]] or [rows, 8192, 4096, 2048, 1024]
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    x = torch.randn(rows, n, device=dev)
    dy = torch.randn(rows, n, device=dev)
    a = 1 + 0.1 * torch.randn(n, device=dev)
    d = 1 + 0.1 * torch.randn(n, device=dev)
    bias = 0.1 * torch.randn(n, device=dev)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    h2 = F.new_h2cache(rows, n, dev)
    grads = [torch.zeros(n, device=dev) for _ in range(3)]
    F.prepare(n, dev)

    def step(m):
        per = h2.numel() // rows
        for k in range(0, rows, m):
            e = min(rows, k + m)
            hc = h2[k * per:e * per]
            F.acdc_forward(x[k:e], a, d, bias, out=y[k:e], h2cache=hc)
            F.acdc_backward(x[k:e], dy[k:e], a, d, *grads, accumulate=k > 0, out=dx[k:e], h2cache=hc)

    ref = None
    for m in chunks:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                step(m)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step(m)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out = [t.clone() for t in (y, dx, *grads)]
        if ref is None:
            ref = out
        diff = [float((o - r).abs().max()) for o, r in zip(out, ref)]
        print(json.dumps({"n": n, "rows": rows, "chunk": m, "ms_per_step": ms, "rows_per_s": rows / ms * 1e3,
                          "frac_20N": rows * 20 * n / (ms * 1e-3) / 6551.4e9, "max_diff_vs_full": diff}), flush=True)


if __name__ == "__main__":
    main()
