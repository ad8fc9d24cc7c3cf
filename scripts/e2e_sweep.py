"""HostPipeline e2e rows/s for several chunk counts / buffer sets (N=4096, B=16384).

usage: python scripts/e2e_sweep.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import functional as F  # noqa: E402

n, B, steps = 4096, 16384, 10
dev = torch.device("cuda", 0)
xh, dyh = torch.randn(B, n).pin_memory(), torch.randn(B, n).pin_memory()
yh, dxh = torch.empty(B, n).pin_memory(), torch.empty(B, n).pin_memory()
gh = torch.empty(3, n).pin_memory()
a, d, b = (torch.randn(n, device=dev) for _ in range(3))
grads = torch.zeros(3, n, device=dev)
for chunks, nbuf, ov, direct in [(4, 2, True, False), (4, 2, True, True), (8, 2, True, True), (4, 2, True, False),
                                 (4, 2, True, True)]:
    if True:
        pipe = F.HostPipeline(n, B, dev, chunks=chunks, nbuf=nbuf, overlap_steps=ov, direct_out=direct)

        def step():
            pipe.step(xh, dyh, yh, dxh, a, d, b, (grads[0], grads[1], grads[2]), accumulate=False)
            gh.copy_(grads, non_blocking=True)

        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        print(f"chunks={chunks} nbuf={nbuf} overlap={ov} direct={direct} rows/s={B * steps / (e0.elapsed_time(e1) / 1e3):.4g}",
              flush=True)
