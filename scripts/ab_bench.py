"""Interleaved A/B timing of kernel variants (different builds of libacdc_b200.so).

usage: python scripts/ab_bench.py [--n 4096] [--rows 16384] [--trials 6] lib_a.so lib_b.so ...

Each trial runs every variant in a fresh subprocess (ACDC_LIB_PATH=...), in
rotating order, timing forward and backward separately with CUDA events over
`--iters` launches; reports the median and min per variant and mode.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, torch
sys.path.insert(0, {root!r})
from paper_1511_05946_b200 import functional as F
n, B, iters = {n}, {rows}, {iters}
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(0)
x = torch.randn(B, n, device=dev, generator=g); dy = torch.randn(B, n, device=dev, generator=g)
a = 1 + 0.1 * torch.randn(n, device=dev, generator=g); d = 1 + 0.1 * torch.randn(n, device=dev, generator=g)
b = 0.1 * torch.randn(n, device=dev, generator=g)
gr = torch.zeros(3, n, device=dev); y = torch.empty_like(x); dx = torch.empty_like(x)
F.prepare(n, dev)
out = {{}}
for mode in ("recompute", "h2cache"):
    hc = F.new_h2cache(B, n, dev) if mode == "h2cache" else None
    f = lambda: F.acdc_forward(x, a, d, b, out=y, h2cache=hc)
    bw = lambda: F.acdc_backward(x, dy, a, d, gr[0], gr[1], gr[2], accumulate=False, out=dx, h2cache=hc)
    try:
        for fn in (f, bw):
            for _ in range(3): fn()
    except ValueError:  # mode not supported by this variant
        continue
    f(); torch.cuda.synchronize()
    res = []
    for fn in (f, bw):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(iters):
            fn() if fn is f else (f(), bw())
        e1.record(); torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / iters)
    fwd, both = res
    out[mode] = {{"fwd_ms": fwd, "bwd_ms": both - fwd, "step_ms": both}}
print(json.dumps(out))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--rows", type=int, default=16384)
    ap.add_argument("--trials", type=int, default=6)
    ap.add_argument("--iters", type=int, default=60)
    args = ap.parse_args()
    code = CHILD.format(root=ROOT, n=args.n, rows=args.rows, iters=args.iters)
    results = {lib: [] for lib in args.libs}
    for trial in range(args.trials):
        order = args.libs[trial % len(args.libs):] + args.libs[: trial % len(args.libs)]
        for lib in order:
            env = dict(os.environ, ACDC_LIB_PATH=os.path.abspath(lib))
            out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            if out.returncode != 0:
                print(lib, "FAILED", out.stderr[-800:], file=sys.stderr)
                continue
            results[lib].append(json.loads(out.stdout.strip().splitlines()[-1]))
    summary = {}
    for lib, runs in results.items():
        s = {}
        for mode in ("recompute", "h2cache"):
            for k in ("fwd_ms", "bwd_ms", "step_ms"):
                vals = [r[mode][k] for r in runs if mode in r]
                if vals:
                    s[f"{mode}.{k}"] = {"median": statistics.median(vals), "min": min(vals)}
        summary[os.path.basename(lib)] = s
        print(os.path.basename(lib), json.dumps({k: round(v["median"], 4) for k, v in s.items()}))
    json.dump(summary, open(os.path.join(ROOT, "gpurun_out", "ab_summary.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
