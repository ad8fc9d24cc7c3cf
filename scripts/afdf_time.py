"""CUDA-event timing of AFDF forward / backward at N (C5 shape by default).

usage: [ACDC_LIB_PATH=variant.so] python scripts/afdf_time.py [N] [rows] [iters]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import functional as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
dev = torch.device("cuda", 0)
x = torch.randn(rows, n, dtype=torch.complex64, device=dev)
dy = torch.randn(rows, n, dtype=torch.complex64, device=dev)
a = ((1 + 0.1 * torch.randn(n, device=dev)) + 0.1j * torch.randn(n, device=dev)).to(torch.complex64)
d = ((1 + 0.1 * torch.randn(n, device=dev)) + 0.1j * torch.randn(n, device=dev)).to(torch.complex64)
ga = torch.zeros(n, dtype=torch.complex64, device=dev)
gd = torch.zeros_like(ga)
y, dx = torch.empty_like(x), torch.empty_like(x)
fwd = lambda: F.afdf_forward(x, a, d, out=y)
bwd = lambda: F.afdf_backward(x, dy, a, d, ga, gd, accumulate=False, out=dx)
out = {}
for name, fn in (("fwd_ms", fwd), ("bwd_ms", bwd)):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    out[name] = round(e0.elapsed_time(e1) / iters, 4)
print(os.path.basename(os.environ.get("ACDC_LIB_PATH", "default")), json.dumps(out))
