"""Minimal HL-kernel calls for compute-sanitizer synccheck (one size per run)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import functional as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dev = torch.device("cuda", 0)
x, dy = torch.randn(3, n, device=dev), torch.randn(3, n, device=dev)
a = torch.ones(n, device=dev)
gr = torch.zeros(3, n, device=dev)
hc = F.new_h2cache(3, n, dev)
F.acdc_forward(x, a, a, a, h2cache=hc)
F.acdc_backward(x, dy, a, a, gr[0], gr[1], gr[2], h2cache=hc)
torch.cuda.synchronize()
print("ok", n)
