"""A few AFDF forward+backward steps at N (C5 shape by default), for ncu.

usage: python scripts/afdf_probe.py [N] [rows]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import functional as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
dev = torch.device("cuda", 0)
x = torch.randn(rows, n, dtype=torch.complex64, device=dev)
dy = torch.randn(rows, n, dtype=torch.complex64, device=dev)
a = (1 + 0.1 * torch.randn(n, device=dev)) + 0.1j * torch.randn(n, device=dev)
d = (1 + 0.1 * torch.randn(n, device=dev)) + 0.1j * torch.randn(n, device=dev)
a, d = a.to(torch.complex64), d.to(torch.complex64)
ga = torch.zeros(n, dtype=torch.complex64, device=dev)
gd = torch.zeros_like(ga)
y, dx = torch.empty_like(x), torch.empty_like(x)
for _ in range(3):
    F.afdf_forward(x, a, d, out=y)
    F.afdf_backward(x, dy, a, d, ga, gd, accumulate=False, out=dx)
torch.cuda.synchronize()
print("ok", n, rows)
