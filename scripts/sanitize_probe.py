"""One small call of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).

Covers: forward (recompute and h2-cache) + TMEM backward (mbarrier bulk copies
of dy into the reused exchange buffer, TMEM alloc/dealloc, cross-group
parking) launched back to back under PDL, the recompute backward, the
two-stage gradient reduction (many row groups at N=128), the SGD-fused
reduction followed by a dependent backward, the fused cascade forward and
its block backwards (ReLU / inverse-perm epilogues, PDL chain; two-block
launches and the deferred multi-block reduction), AFDF forward
and backward, the complex FFT and the DCT / IDCT kernels.
usage: python scripts/sanitize_probe.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import AcdcLayer, Cascade, PermutationLayer, ReluLayer  # noqa: E402
from paper_1511_05946_b200 import functional as F  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
rn = lambda *s: torch.randn(*s, device=dev, generator=g)


def layer(n, rows, cache):
    x, dy = rn(rows, n), rn(rows, n)
    a, d, b = 1 + 0.1 * rn(n), 1 + 0.1 * rn(n), 0.1 * rn(n)
    gr = torch.zeros(3, n, device=dev)
    hc = F.new_h2cache(rows, n, dev) if cache else None
    for _ in range(2):  # back to back: PDL forward -> backward -> reduction -> next forward
        y = F.acdc_forward(x, a, d, b, h2cache=hc)
        F.acdc_backward(x, y if cache else dy, a, d, gr[0], gr[1], gr[2], h2cache=hc)


layer(1024, 12, True)     # TMEM backward (2 groups per CTA), odd row pairs per group
layer(4096, 7, True)      # TMEM backward at the metric size, a ragged last pair
layer(4096, 6, False)     # recompute backward
layer(128, 2100, False)   # two-stage reduction (many row groups)
layer(16384, 3, True)     # half-length plan (N/2-point FFT per row), TMEM accumulators
layer(32768, 2, True)     # half-length plan, tables in global memory, grad_a partial in global memory
layer(8192, 5, False)     # half-length recompute backward
layer(2048, 9, True)      # half-length plan at its smallest size (the metric path's kernels, N/2 = 1024)
# SGD-fused reduction, then a backward of the same layer (PDL ordering)
n, rows = 1024, 10
x, dy = rn(rows, n), rn(rows, n)
a, d, b = 1 + 0.1 * rn(n), 1 + 0.1 * rn(n), torch.zeros(n, device=dev)
vel = [torch.zeros(n, device=dev) for _ in range(3)]
hc = F.new_h2cache(rows, n, dev)
F.acdc_forward(x, a, d, b, h2cache=hc)
for _ in range(2):
    F.acdc_backward_sgd(x, dy, (a, d, b), vel, (0.1,) * 3, (0.0,) * 3, 0.9, h2cache=hc)
# fused cascade (ReLU + Perm epilogues)
rng = np.random.default_rng(0)
ls = []
for i in range(3):
    L = AcdcLayer(512, device=dev)
    L.a.normal_(1.0, 0.1)
    ls.append(L)
    if i < 2:
        ls += [ReluLayer(512, device=dev), PermutationLayer(512, perm=rng.permutation(512), device=dev)]
c = Cascade(ls)
c.forward(rn(9, 512))
c.backward(rn(9, 512))  # two-block backward (block pairs 2+1), block 0 alone, one multi-block reduction
c.forward(rn(9, 512))
c.backward(rn(9, 512), on_layer=lambda layer: None)  # per-block gather backward + reduction (hook path)
# 4-block stack at N=1024 without permutations: two two-block launches, deferred reduction
ls = [AcdcLayer(1024, device=dev) for _ in range(4)]
c = Cascade(ls)
c.forward(rn(7, 1024))
c.backward(rn(7, 1024))
# ACDC-only stack at N=4096: half-length fused cascade (parameter re-layout, blocks chained in registers),
# deferred half-length block backwards, then the per-block path (hook)
ls = [AcdcLayer(4096, device=dev) for _ in range(3)]
c = Cascade(ls)
c.forward(rn(5, 4096))
c.backward(rn(5, 4096))
c.forward(rn(5, 4096))
c.backward(rn(5, 4096), on_layer=lambda layer: None)
# AFDF, FFT, DCT
for n in (256, 8192):
    z = torch.complex(rn(5, n), rn(5, n))
    a = torch.complex(1 + 0.1 * rn(n), 0.1 * rn(n))
    ga, gd = torch.zeros(n, dtype=torch.complex64, device=dev), torch.zeros(n, dtype=torch.complex64, device=dev)
    y = F.afdf_forward(z, a, a)
    F.afdf_backward(z, y, a, a, ga, gd)
    F.fft(z)
    F.ifft(z)
F.dct(rn(3, 4096))
F.idct(rn(3, 4096))
torch.cuda.synchronize()
print("sanitize probe ok")


# fused small-batch step: one cluster of CTAs, gradients over distributed shared memory
def step(n, rows):
    x, dy = rn(rows, n), rn(rows, n)
    a, d, b = 1 + 0.1 * rn(n), 1 + 0.1 * rn(n), 0.1 * rn(n)
    gr = torch.zeros(3, n, device=dev)
    for _ in range(2):
        F.acdc_step(x, dy, a, d, b, gr[0], gr[1], gr[2])


step(256, 128)   # C1: 4 CTAs
step(256, 1000)  # full cluster, several row pairs per group, ragged last pair
step(4096, 9)    # one group per CTA
torch.cuda.synchronize()
print("sanitize probe: fused step done")
