"""PCIe ceilings for the e2e path: pinned H2D, D2H and both at once, plus the
HostPipeline at several chunk counts (N=4096, 16384 rows, fp32).

usage: python scripts/pcie_probe.py
"""

from __future__ import annotations

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    dev = torch.device("cuda", 0)
    n, rows = 4096, 16384
    nb = 2 * rows * n * 4  # two [rows, n] fp32 tensors each way
    h_in = torch.empty(2, rows, n, pin_memory=True).normal_()
    h_out = torch.empty(2, rows, n, pin_memory=True)
    d_in = torch.empty(2, rows, n, device=dev)
    d_out = torch.empty(2, rows, n, device=dev).normal_()
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {}
    res["h2d_GBps"] = nb / timed(lambda: d_in.copy_(h_in, non_blocking=True)) / 1e6
    res["d2h_GBps"] = nb / timed(lambda: h_out.copy_(d_out, non_blocking=True)) / 1e6

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    ms = timed(both)
    res["both_ms"] = ms
    res["both_GBps_each"] = nb / ms / 1e6

    for chunk_mb in (4, 16, 64):
        ce = chunk_mb * (1 << 20) // 4
        fi, fo = h_in.view(-1), h_out.view(-1)
        gi, go = d_in.view(-1), d_out.view(-1)

        def chunked():
            cur = torch.cuda.current_stream()
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            for o in range(0, fi.numel(), ce):
                with torch.cuda.stream(s1):
                    gi[o:o + ce].copy_(fi[o:o + ce], non_blocking=True)
                with torch.cuda.stream(s2):
                    fo[o:o + ce].copy_(go[o:o + ce], non_blocking=True)
            cur.wait_stream(s1)
            cur.wait_stream(s2)

        res[f"both_chunk{chunk_mb}MB_GBps_each"] = nb / timed(chunked) / 1e6

    from paper_1511_05946_b200 import functional as F

    a = 1 + 0.1 * torch.randn(n, device=dev)
    d = 1 + 0.1 * torch.randn(n, device=dev)
    b = 0.1 * torch.randn(n, device=dev)
    grads = tuple(torch.zeros(n, device=dev) for _ in range(3))
    for chunks, nbuf, ramp, direct in ((8, 2, False, False), (16, 3, True, False), (8, 2, False, True),
                                       (16, 3, True, True), (32, 3, True, True), (4, 2, False, True)):
        pipe = F.HostPipeline(n, rows, dev, chunks=chunks, nbuf=nbuf, ramp=ramp, direct_out=direct)
        ms = timed(lambda: pipe.step(h_in[0], h_in[1], h_out[0], h_out[1], a, d, b, grads), iters=5)
        res[f"pipeline_c{chunks}_b{nbuf}_r{int(ramp)}_d{int(direct)}_ms"] = ms
        del pipe
        torch.cuda.empty_cache()
    # the pipeline's stream/event structure with the kernels removed
    pipe = F.HostPipeline(n, rows, dev, chunks=16, nbuf=3, ramp=True)
    real_f, real_b = F.acdc_forward, F.acdc_backward
    F.acdc_forward = lambda *args, **kw: None
    F.acdc_backward = lambda *args, **kw: None
    try:
        res["pipeline_copy_only_ms"] = timed(lambda: pipe.step(h_in[0], h_in[1], h_out[0], h_out[1], a, d, b, grads))
    finally:
        F.acdc_forward, F.acdc_backward = real_f, real_b
    del pipe
    # per-chunk timeline of one step (ms from the step start): upload done,
    # compute done, download done
    pipe = F.HostPipeline(n, rows, dev, chunks=16, nbuf=3, ramp=True, direct_out=True)
    pipe.step(h_in[0], h_in[1], h_out[0], h_out[1], a, d, b, grads)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    ev = pipe.step(h_in[0], h_in[1], h_out[0], h_out[1], a, d, b, grads, timeline=True)
    torch.cuda.synchronize()
    res["timeline"] = [[round(t0.elapsed_time(e), 3) for e in trip] for trip in ev]
    res["timeline_rows"] = [hi - lo for lo, hi in pipe.spans]
    # direct_out correctness against the staged pipeline
    p1 = F.HostPipeline(n, rows, dev, chunks=8, direct_out=False)
    p2 = F.HostPipeline(n, rows, dev, chunks=8, direct_out=True)
    o1 = torch.empty(2, rows, n, pin_memory=True)
    o2 = torch.empty(2, rows, n, pin_memory=True)
    g1 = tuple(torch.zeros(n, device=dev) for _ in range(3))
    g2 = tuple(torch.zeros(n, device=dev) for _ in range(3))
    p1.step(h_in[0], h_in[1], o1[0], o1[1], a, d, b, g1)
    p2.step(h_in[0], h_in[1], o2[0], o2[1], a, d, b, g2)
    torch.cuda.synchronize()
    res["direct_equal"] = bool(torch.equal(o1, o2)) and all(torch.equal(u, v) for u, v in zip(g1, g2))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
