"""Run a few fwd+bwd steps of one ACDC layer at size N (for ncu launch lists).

usage: python scripts/size_probe.py N [rows] [mode]
"""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1511_05946_b200 import functional as F  # noqa: E402

n = int(sys.argv[1])
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
mode = sys.argv[3] if len(sys.argv) > 3 else ("h2cache" if F.h2cache_supported(n) else "recompute")
dev = torch.device("cuda", 0)
x = torch.randn(rows, n, device=dev)
dy = torch.randn(rows, n, device=dev)
a, d, b = (torch.randn(n, device=dev) for _ in range(3))
g = torch.zeros(3, n, device=dev)
hc = F.new_h2cache(rows, n, dev) if mode == "h2cache" else None
F.prepare(n, dev)
for _ in range(3):
    F.acdc_forward(x, a, d, b, h2cache=hc)
    F.acdc_backward(x, dy, a, d, g[0], g[1], g[2], accumulate=False, h2cache=hc)
torch.cuda.synchronize()
print("ok", n, rows, mode)
