"""A few steps of the C4 deep cascade (32 ACDC layers, N=4096) or C3, for ncu launch lists.

usage: python scripts/cascade_probe.py [c4|c3]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import AcdcLayer, Cascade, PermutationLayer, ReluLayer  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
n, depth, B, rp = (4096, 32, 4096, False) if which == "c4" else (1024, 12, 8192, True)
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
layers = []
for i in range(depth):
    L = AcdcLayer(n, device=dev)
    L.a.normal_(1.0, 0.061)
    L.d.normal_(1.0, 0.061)
    layers.append(L)
    if rp and i < depth - 1:
        layers += [ReluLayer(n, device=dev), PermutationLayer(n, perm=rng.permutation(n), device=dev)]
casc = Cascade(layers)
x = torch.randn(B, n, device=dev)
dy = torch.randn(B, n, device=dev)
for _ in range(2):
    casc.forward(x)
    casc.backward(dy)
torch.cuda.synchronize()
print("ok", which, casc.fused)
