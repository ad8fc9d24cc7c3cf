"""Forward / backward parity of the loaded library at one size vs the fp64 oracle
(test tooling for single-size A/B builds: ACDC_LIB_PATH=variant.so python tests/variant_check.py N rows)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import acdc_oracle as O  # noqa: E402  (checker only)
from paper_1511_05946_b200 import functional as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 37
rng = np.random.default_rng(1)
f = lambda *s, m=0.0, sd=1.0: (m + sd * rng.standard_normal(s)).astype(np.float32)
x, dy = f(rows, n), f(rows, n)
a, d, b = f(n, m=1.0, sd=0.3), f(n, m=1.0, sd=0.3), f(n, sd=0.3)
dev = torch.device("cuda", 0)
t = lambda v: torch.as_tensor(v, device=dev)
X, DY, A, D, B = (v.astype(np.float64) for v in (x, dy, a, d, b))
yr, h2 = O.acdc_forward(X, A, D, B)
dxr, gar, gdr, gbr = O.acdc_backward(X, h2, DY, A, D)
for mode in ("recompute", "h2cache"):
    hc = F.new_h2cache(rows, n, dev) if mode == "h2cache" else None
    try:
        y = F.acdc_forward(t(x), t(a), t(d), t(b), h2cache=hc)
    except ValueError as e:  # mode not supported by this variant
        print(mode, "skipped:", e)
        continue
    g = [torch.zeros(n, device=dev) for _ in range(3)]
    dx = F.acdc_backward(t(x), t(dy), t(a), t(d), *g, accumulate=False, h2cache=hc)
    torch.cuda.synchronize()
    errs = {
        "y": float(np.abs(y.double().cpu().numpy() - yr).max()) / O.fp32_tolerance(n, yr),
        "dx": float(np.abs(dx.double().cpu().numpy() - dxr).max()) / O.fp32_tolerance(n, dxr),
    }
    for nm, mine, ref in zip(("ga", "gd", "gb"), g, (gar, gdr, gbr)):
        errs[nm] = float(np.abs(mine.double().cpu().numpy() - ref).max()) / O.grad_tolerance(n, rows, ref)
    print(mode, "err/tol", {k: round(v, 3) for k, v in errs.items()}, "OK" if max(errs.values()) <= 1 else "FAIL")
