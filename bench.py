"""Benchmark: fused ACDC forward+backward rows/s at N=4096 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU, NCCL)

A step is one pass of the hot path over one batch through the reference-shaped
layer API: ``AcdcLayer.forward`` (y = C3(d*C2(a*x)+b)), ``AcdcLayer.backward``
(dx and the three diagonal gradients, accumulated), the fixed-order gradient
reduction, and ``DataParallel.allreduce_grads`` (for N > 1 one NCCL all-reduce
of the flat [ga|gd|gb] gradient buffer).  Batch 16384 rows per GPU (weak
scaling, the default) or 16384 rows in total (``--scaling strong``).  Inputs
are synthetic Gaussian fp32 tensors resident in HBM (each 256 MiB > the
126 MB L2, so no L2 flush is needed between steps).

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (one process per GPU, NCCL).

Roofline: algorithmic bytes per row are 8N for the forward,
12N for the backward (x, dy in, dx out) and 20N per step; the h2 cache the
kernels may keep (+4N out, +4N in) is reported as moved bytes, not counted.

``--impl reference`` times the reference's own compiled CPU kernels
(``oracle/_ref``, the Cython ``_kernels.pyx`` built from /root/reference) on
this host's cores for the same metric, on a bounded row sample per step.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_FEAT = 4096
BATCH = 16384
METRIC = "ACDC fwd+bwd rows/sec at N=4096 (1/2/4/8 B200), % of HBM roofline"
UNIT = "rows/s"
BYTES_FWD = 8 * N_FEAT  # x in, y out (fp32)
BYTES_BWD = 12 * N_FEAT  # x, dy in, dx out (h2 recomputed)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_FEAT)
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager steps instead of replays of the step captured in a CUDA graph")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: --batch rows per GPU; strong: --batch rows in total, sharded over the ranks")
    ap.add_argument("--mode", default="auto", choices=["auto", "recompute", "h2cache"],
                    help="recompute h2 in the backward (PAPER.md:275) or cache it from the forward "
                         "(layers.py:145); auto times both and reports the faster")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during timing."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._pump, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "power_w_max": max(power) if power else None,
            "samples": len(sm),
            "reasons": sorted(reasons),
        }


# ------------------------------------------------------------- CPU baseline
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_cpu(n, threads, rows, seconds=None, steps=None, warmup=0):
    """Time the reference's compiled kernels (oracle/_ref) on host threads.

    Returns (rows_per_s, kind, sample_desc, per_step_times)."""
    from oracle import ref_kernels

    rng = np.random.default_rng(0)
    a, d = 1 + 0.1 * rng.standard_normal((2, n))
    bias = 0.1 * rng.standard_normal(n)
    x = rng.standard_normal((rows, n))
    dy = rng.standard_normal((rows, n))
    if ref_kernels.load() is not None:
        layer = ref_kernels.RefAcdc(a, d, bias)
        kind = "reference"

        def step():
            ref_kernels.fwd_bwd_threaded(layer, x, dy, threads)
    else:  # the numpy restatement (fp64) as a port
        from oracle import acdc_oracle as O

        kind = "port"
        threads = 1

        def step():
            y, h2 = O.acdc_forward(x, a, d, bias)
            O.acdc_backward(x, h2, dy, a, d)
    for _ in range(warmup):
        step()
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
        if steps is not None and len(times) >= steps:
            break
        if steps is None and time.perf_counter() - t_start >= seconds:
            break
    total = sum(times)
    rps = rows * len(times) / total
    sample = (f"{len(times)} x fwd+bwd of {rows} rows at N={n}, fp64 (reference dtype), "
              f"{threads} host threads, {cpu_model()}")
    return rps, kind, sample, times, threads


# ------------------------------------------------------------------ our arm
def free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(gpus: int, script: str) -> None:
    """``--gpus N`` (N > 1) outside torchrun: re-run this script under
    ``torch.distributed.run`` with N ranks on this node and exit with its code
    (rank 0 prints the JSON line)."""
    if gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(script), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def dist_setup(gpus):
    """One process per GPU.  ``ACDC_DIST_BACKEND=gloo`` + ``ACDC_SHARE_GPU=1``
    put every rank on cuda:0 (exercises the multi-rank path on a 1-GPU box;
    NCCL refuses two ranks on one device)."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if gpus > 1 and world != gpus:
        raise SystemExit(f"--gpus {gpus} but WORLD_SIZE={world}")
    if world > 1:
        share = os.environ.get("ACDC_SHARE_GPU") == "1"
        ndev = torch.cuda.device_count()
        if not share and world > ndev:
            raise SystemExit(f"{world} ranks but only {ndev} visible GPUs")
        dev = 0 if share else local
        torch.cuda.set_device(dev)
        backend = os.environ.get("ACDC_DIST_BACKEND", "nccl")
        kw = {"device_id": torch.device("cuda", dev)} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
        local = dev
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(v, world):
    import torch
    import torch.distributed as dist

    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1511_05946_b200 import AcdcLayer, _lib, functional as F
    from paper_1511_05946_b200.parallel import DataParallel, shard_rows

    world, rank, local = dist_setup(args.gpus)
    n = args.n
    if args.scaling == "strong":  # --batch rows in total, contiguous shards
        lo, hi = shard_rows(args.batch, world, rank)
        B = hi - lo
        global_rows = args.batch
    else:
        B = args.batch
        global_rows = B * world
    dev = torch.device("cuda", torch.cuda.current_device())
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = torch.randn(B, n, device=dev, generator=g)
    dy = torch.randn(B, n, device=dev, generator=g)
    g.manual_seed(99)  # replicated parameters: the same seed on every rank
    a = 1 + 0.1 * torch.randn(n, device=dev, generator=g)
    d = 1 + 0.1 * torch.randn(n, device=dev, generator=g)
    bias = 0.1 * torch.randn(n, device=dev, generator=g)
    F.prepare(n, dev)
    stream = torch.cuda.current_stream()

    def make(mode):
        """The reference-shaped layer (layers.py:108-156) wrapped for data
        parallelism: grads live in one flat buffer, one all-reduce per step."""
        layer = AcdcLayer(n, device=dev, cache_h2=(mode == "h2cache"))
        layer.a.copy_(a)
        layer.d.copy_(d)
        layer.bias_d.copy_(bias)
        return DataParallel(layer)

    def timed(mode):
        """W warm-up + exactly K timed steps of one mode; per-kernel CUDA events."""
        dp = make(mode)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]

        def step(i=None):
            e = ev[i] if i is not None else None
            dp.zero_grads()
            if e: e[0].record(stream)
            dp.forward(x)
            if e: e[1].record(stream)
            dp.backward(dy)
            if e: e[2].record(stream)
            dp.allreduce_grads()
            if e: e[3].record(stream)

        for _ in range(max(args.warmup, 3)):
            step()
        for i in range(args.steps):  # per-kernel split (eager, events between the kernels): before
            step(i)                  # the capture, so the eager steps reuse the warm-up's allocations
        torch.cuda.synchronize()
        # the whole step (zero grads, forward, backward + reduction, all-reduce)
        # captured once and replayed (SURVEY §8(d) timing; removes the per-kernel
        # host launch cost); the captured kernels keep their programmatic
        # dependent launches.  Eager steps if capture is not possible.
        run, graph_note = step, "eager steps"
        if not args.no_graph:
            try:
                side = torch.cuda.Stream()
                side.wait_stream(stream)
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.stream(side):
                    step()
                    torch.cuda.synchronize()
                    with torch.cuda.graph(graph, stream=side):
                        step()
                torch.cuda.synchronize()
                for _ in range(2):
                    graph.replay()
                run, graph_note = graph.replay, "CUDA-graph replay of the whole step"
            except Exception as e:  # noqa: BLE001 (timed eagerly instead)
                print(f"bench: CUDA-graph capture failed ({e}); timing eager steps", file=sys.stderr)
                torch.cuda.synchronize()
        barrier(world)
        sampler = ClockSampler(local)
        sampler.start()
        time.sleep(0.15)
        barrier(world)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):  # no events between the kernels: they would break the
            run()                    # forward -> backward programmatic dependent launch
        t1.record(stream)
        barrier(world)
        clocks = sampler.stop()
        max_ms = max_over_ranks(t0.elapsed_time(t1), world)
        res = {
            "mode": mode,
            "max_ms": max_ms,
            "fwd_ms": sum(e[0].elapsed_time(e[1]) for e in ev) / args.steps,
            "bwd_ms": sum(e[1].elapsed_time(e[2]) for e in ev) / args.steps,
            "ar_ms": sum(e[2].elapsed_time(e[3]) for e in ev) / args.steps,
            "clocks": clocks,
            "value": global_rows * args.steps / (max_ms / 1e3),
            "grads_finite": bool(torch.isfinite(dp.flat).all()),
            "timing": graph_note,
        }
        del dp
        torch.cuda.empty_cache()
        return res

    modes = ["recompute"] if (not F.h2cache_supported(n) or args.mode == "recompute") else (
        ["h2cache"] if args.mode == "h2cache" else ["recompute", "h2cache"])
    runs = [timed(m) for m in modes]
    best = max(runs, key=lambda r: r["value"])
    other = [r for r in runs if r is not best]
    fwd_ms, bwd_ms, ar_ms, clocks = best["fwd_ms"], best["bwd_ms"], best["ar_ms"], best["clocks"]
    max_ms = best["max_ms"]
    ms_per_step = max_ms / args.steps
    value = best["value"]
    # algorithmic bytes per row: fwd 8N, bwd 12N; the h2 cache adds 4N out + 4N in (moved, not counted)
    cache_b = 4 * n if best["mode"] == "h2cache" else 0
    alg_fwd, alg_bwd = 8 * n, 12 * n
    mov_fwd, mov_bwd = alg_fwd + cache_b, alg_bwd + cache_b

    # e2e through the public API with host buffers (pinned), copies in the timed region
    e2e = None
    if not args.no_e2e:
        e2e = e2e_measure(F, n, B, a, d, bias, dev, world, steps=max(3, min(args.steps, 10)),
                          h2cache=best["mode"] == "h2cache", global_rows=global_rows)

    dense = None
    if not args.no_dense and rank == 0:
        dense = dense_measure(n, B, dev)

    out = None
    if rank == 0:
        hbm, src = peaks()
        # dominant kernel = the longer of fwd / bwd (bwd: backward kernel + grad reduce).  Which
        # kernels run: the half-length plan for 1024 <= n <= 32768 (hl_kernels.cu ACDC_HL_MIN_LOGN,
        # off with ACDC_HL=0), else the row-pair kernels, whose h2-cache backward is the TMEM kernel
        # for 512 <= n (acdc_kernels.cu bwd_tm_ok)
        hl = 1024 <= n <= 32768 and os.environ.get("ACDC_HL", "1") != "0"
        if bwd_ms >= fwd_ms:
            if hl:
                bk = "acdc_bwd_hl_kernel"
            else:
                bk = "acdc_bwd_tm_kernel" if (best["mode"] == "h2cache" and 512 <= n) else "acdc_bwd_kernel"
            kname, kms, kalg, kmov = f"{bk}(+grad_reduce)", bwd_ms, alg_bwd * B, mov_bwd * B
        else:
            kname, kms, kalg, kmov = ("acdc_fwd_hl_kernel" if hl else "acdc_fwd_kernel"), fwd_ms, alg_fwd * B, mov_fwd * B
        achieved = kalg / (kms / 1e3) / 1e9
        step_alg = (alg_fwd + alg_bwd) * B
        step_gbs = step_alg / (ms_per_step / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            try:
                t = json.load(open(tpath)).get(kname.split("(")[0])
                traffic = t * B / 16384 if (t is not None and n == N_FEAT) else None
            except Exception:
                traffic = None
        out = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(args.warmup, 3),
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic Gaussian x, dy ~ N(0,1); a, d ~ N(1, 0.1^2); bias ~ N(0, 0.1^2)",
            "config": {
                "workload": f"single ACDC layer fwd+bwd (AcdcLayer under DataParallel), N={n}, "
                            + (f"batch {B} rows per GPU" if args.scaling == "weak" else f"batch {args.batch} in total")
                            + ", fp32",
                "n": n,
                "rows_per_gpu": B,
                "global_rows": global_rows,
                "parallelism": f"dp{world}" if world > 1 else "single",
                "l2": "inputs larger than L2 (x, dy, y, dx are 256 MiB each at B=16384); no flush",
                "step_timing": best["timing"],
            },
            "roofline": {
                "kernel": kname,
                "bound": "hbm",
                "achieved": achieved,
                "peak": hbm,
                "peak_source": src,
                "unit": "GB/s",
                "frac": achieved / hbm,
                "traffic": traffic,
                "algorithmic_bytes_per_launch": kalg,
                "algorithmic_bytes_per_row": kalg // B,
                "moved_bytes_per_launch": kmov,
                "moved_frac": kmov / (kms / 1e3) / 1e9 / hbm,
                "traffic_over_algorithmic": (traffic / kalg) if traffic else None,
                "avg_launch_ms": kms,
                "timing": "CUDA events around each kernel over K eager steps right before the timed loop "
                          "(events between the kernels inside the timed loop would break the forward -> "
                          "backward programmatic dependent launch)",
            },
            "mode": best["mode"],
            "other_modes": [{k: r[k] for k in ("mode", "value", "fwd_ms", "bwd_ms")} for r in other],
            "roofline_step": {
                "bytes_per_row": alg_fwd + alg_bwd,
                "bytes_moved_per_row": mov_fwd + mov_bwd,
                "achieved_gbs": step_gbs,
                "frac": step_gbs / hbm,
                "fwd_ms": fwd_ms,
                "bwd_ms": bwd_ms,
                "allreduce_ms": ar_ms,
            },
            "clocks": clocks,
            # our kernels per step: fwd + bwd + its one- or two-stage grad reduction (the zero_grads
            # memset is torch's, not counted)
            "gpu_launches": (1 + _lib.load().acdc_bwd_launch_count(B, n, 1 if best["mode"] == "h2cache" else 0))
            * args.steps,
            "grads_finite": best["grads_finite"],
            "e2e": e2e,
            "dense_cublas": dense,
        }
        if not args.no_cpu_baseline and world == 1:
            thr = cpu_threads()
            rows = max(1024, 64 * thr)
            rps, kind, sample, _, used = reference_cpu(n, thr, rows, seconds=12.0, warmup=1)
            out["cpu_baseline"] = {"value": rps, "unit": UNIT, "cores": used, "kind": kind, "sample": sample}
    if world > 1:
        dist.destroy_process_group()
    return out


def e2e_measure(F, n, B, a, d, bias, dev, world, steps, h2cache=False, global_rows=None):
    """Rows/s through the public API with pinned HOST buffers: per step the
    host->device copy of x and dy, forward, backward, and the device->host
    copy of y, dx and the gradients are all inside the timed region.  Uses
    functional.HostPipeline (chunked, three streams: upload / kernels /
    download overlap on the full-duplex PCIe link)."""
    import torch
    import torch.distributed as dist

    xh = torch.randn(B, n).pin_memory()
    dyh = torch.randn(B, n).pin_memory()
    yh = torch.empty(B, n).pin_memory()
    dxh = torch.empty(B, n).pin_memory()
    gh = torch.empty(3, n).pin_memory()
    grads = torch.zeros(3, n, device=dev)
    pipe = F.HostPipeline(n, B, dev, chunks=4, h2cache=h2cache)  # scripts/e2e_sweep.py

    def step():
        pipe.step(xh, dyh, yh, dxh, a, d, bias, (grads[0], grads[1], grads[2]), accumulate=False)
        if world > 1:
            dist.all_reduce(grads)
        gh.copy_(grads, non_blocking=True)

    step()
    barrier(world)
    s = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(s)
    for _ in range(steps):
        step()
    t1.record(s)
    barrier(world)
    ms = max_over_ranks(t0.elapsed_time(t1), world)
    return {
        "value": (global_rows or world * B) * steps / (ms / 1e3),
        "unit": UNIT,
        "h2d_bytes_per_step": 2 * B * n * 4,
        "d2h_bytes_per_step": 2 * B * n * 4 + 3 * n * 4,
        "steps": steps,
        "path": "functional.HostPipeline (C ABI kernels; pinned host x, dy -> y, dx, grads; 4 chunks, 3 streams, "
                "uploads of a step overlap the previous step's downloads)",
    }


def dense_measure(n, B, dev):
    """cuBLAS dense linear of the same N, fwd + bwd (dX and dW), fp32, TF32 off and on."""
    import torch

    res = {}
    w = torch.randn(n, n, device=dev) / math.sqrt(n)
    x = torch.randn(B, n, device=dev)
    gy = torch.randn(B, n, device=dev)
    for tf32 in (False, True):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        def step():
            y = x @ w
            gx = gy @ w.t()
            gw = x.t() @ gy
            return y, gx, gw
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res["tf32" if tf32 else "fp32"] = {"rows_per_s": B / (ms / 1e3), "ms_per_step": ms,
                                            "tflops": 6 * B * n * n / (ms / 1e3) / 1e12}
    torch.backends.cuda.matmul.allow_tf32 = False
    return res


def run_reference(args):
    """The reference's own compiled CPU kernels (oracle/_ref: _kernels.pyx built
    from /root/reference) driven with the reference layer's call sequence
    (layers.py:141-156), rows sharded over all host threads.  Each step is the
    full batch when the whole run fits in ~3 minutes at the measured rate,
    else a contiguous row sample of it (CPU rows/s does not depend on the batch
    size at N=4096: every row is an independent transform pair)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    thr = cpu_threads()
    full = args.batch * (world if args.scaling == "weak" else 1)
    rate, _, _, _, _ = reference_cpu(args.n, thr, max(512, 32 * thr), steps=1, warmup=1)  # calibration
    budget_s = 150.0
    rows = int(min(full, max(512, rate * budget_s / max(1, args.steps + args.warmup))))
    rows -= rows % 2
    rps, kind, sample, times, used = reference_cpu(args.n, thr, rows, steps=args.steps, warmup=args.warmup)
    ms = 1e3 * sum(times) / len(times)
    return {
        "metric": METRIC,
        "value": rps,
        "unit": UNIT,
        "impl": "reference",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic Gaussian",
        "config": {"workload": f"single ACDC layer fwd+bwd, N={args.n}, reference CPU path, "
                               f"{rows} of the {full} rows per step" + (" (full batch)" if rows == full else
                                                                        " (row sample; rows/s is batch-invariant)"),
                   "n": args.n, "rows_per_step": rows, "batch": full,
                   "tables": "Makhoul tables from oracle.acdc_oracle.tables (transforms.py:86-122 restated, pinned "
                             "against the reference's golden vectors)"},
        "cpu_baseline": {"value": rps, "unit": UNIT, "cores": used, "kind": kind, "sample": sample},
        "e2e": {"value": rps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    maybe_spawn(args.gpus, __file__)
    if args.impl == "reference":
        out = run_reference(args)
    else:
        out = run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
