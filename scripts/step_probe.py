"""Graph-replayed fwd+bwd step time (h2-cache mode where supported) for a list
of (n, rows) shapes; one JSON line per shape.  Used for A/B runs of launch
policies (e.g. ACDC_GRID_SPREAD=0/1).

  python scripts/step_probe.py n:rows [n:rows ...]
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from c1_probe import graph_us  # noqa: E402
from paper_1511_05946_b200 import functional as F  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for spec in sys.argv[1:]:
        n, rows = (int(v) for v in spec.split(":"))
        F.prepare(n, dev)
        x = torch.randn(rows, n, device=dev)
        dy = torch.randn(rows, n, device=dev)
        a, d, b = (torch.randn(n, device=dev) for _ in range(3))
        g = torch.zeros(3, n, device=dev)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        hc = F.new_h2cache(rows, n, dev) if F.h2cache_supported(n) else None
        fwd = lambda: F.acdc_forward(x, a, d, b, out=y, h2cache=hc)  # noqa: E731
        bwd = lambda: F.acdc_backward(x, dy, a, d, g[0], g[1], g[2], accumulate=False, out=dx, h2cache=hc)  # noqa: E731
        reps = 2000 if rows * n <= (1 << 22) else 200
        us = graph_us(lambda: (fwd(), bwd()), reps)
        print(json.dumps({"n": n, "rows": rows, "spread": os.environ.get("ACDC_GRID_SPREAD", "1"), "step_us": us,
                          "frac_20N": rows * 20 * n / (us * 1e-6) / 6551.4e9}), flush=True)


if __name__ == "__main__":
    main()
