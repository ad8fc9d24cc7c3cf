"""Probe: our row FFT engine (acdc_fft_c64 -> fft_rows_kernel) against cuFFT
(torch.fft.fft) on batched complex64 rows, at batch sizes that stay in L2
(compute-bound) and that stream from HBM.  CUDA-graph replay, CUDA events.

  python scripts/fft_vs_cufft.py [n]
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import functional as F  # noqa: E402


def timed(fn, reps=50):
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
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    dev = torch.device("cuda", 0)
    F.prepare(n, dev)
    for rows in (256, 512, 1024, 2048, 8192, 32768):
        z = torch.randn(rows, n, dtype=torch.complex64, device=dev)
        out = torch.empty_like(z)
        ours = timed(lambda: F._fft_rows(z, False, out=out))
        cu = timed(lambda: torch.fft.fft(z, out=out))
        err = float((F._fft_rows(z, False) - torch.fft.fft(z)).abs().max())
        byt = rows * n * 16
        print(json.dumps({"n": n, "rows": rows, "ours_us": ours * 1e3, "cufft_us": cu * 1e3,
                          "ours_fft_per_s": rows / ours * 1e3, "cufft_fft_per_s": rows / cu * 1e3,
                          "ours_gbs": byt / ours / 1e6, "cufft_gbs": byt / cu / 1e6, "max_diff": err}), flush=True)


if __name__ == "__main__":
    main()
