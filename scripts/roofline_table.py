"""Per-kernel roofline table from ncu raw CSV exports (profiles/round2/ncu/raw_*.csv).

usage: python scripts/roofline_table.py [raw_dir] > profiles/round2/roofline.md

For every captured launch: duration, DRAM bytes (read + write), the
ALGORITHMIC bytes of that launch (forward 8N B/row, backward
12N B/row, fp32; AFDF complex64 16N / 24N B/row; cascade forward 8N B/row for
the whole stack; reductions and tables O(N) and not counted) and
achieved = algorithmic / duration against the measured HBM peak
(MEASURED_PEAKS.json), plus traffic / algorithmic (> 1: re-reads or the
h2 cache's extra 4N + 4N).  ncu times are cold-cache and serialised: the
per-kernel shares, not the absolute step time, are what the bench agrees with.
"""

import csv
import glob
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# probe name -> (n, rows, complex) as run by scripts/gpu_r2c.sh
PROBES = {
    "m_cache": (4096, 16384, False), "m_recompute": (4096, 16384, False), "n128": (128, 16384, False),
    "n8192": (8192, 16384, False), "n16384": (16384, 16384, False), "n32768": (32768, 4096, False),
    "c3": (1024, 8192, False), "c5": (8192, 8192, True), "n1024": (1024, 16384, False),
    "n2048": (2048, 16384, False), "n256": (256, 16384, False),
}


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def time_scale(u):
    return {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}.get(u, 1e-6)


def alg_bytes(kname, n, rows, cplx):
    e = 8 if cplx else 4
    if "grad" in kname:
        return None
    if "cascade_fwd" in kname:
        return 2 * e * n * rows
    if "bwd_tm2" in kname:  # two block backwards per launch
        return 2 * 3 * e * n * rows
    if "fwd" in kname:
        return 2 * e * n * rows
    if "bwd" in kname:
        return 3 * e * n * rows
    if "fft_rows" in kname:
        return 2 * 8 * n * rows
    return None


def main():
    raw_dir = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "round2", "ncu")
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        src = "measured"
    except Exception:
        peak, src = 6650.0, "fallback"
    print(f"# Per-kernel HBM roofline (ncu --set full, cold cache; peak {peak:.0f} GB/s, {src})\n")
    print("| probe | kernel | grid x block | regs | duration | DRAM bytes | algorithmic bytes | achieved GB/s | "
          "frac of peak | traffic / algorithmic | issue active % | FMA pipe % | spill loads |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for path in sorted(glob.glob(os.path.join(raw_dir, "raw_*.csv"))):
        probe = re.sub(r"^raw_|\.csv$", "", os.path.basename(path))
        n, rows, cplx = PROBES.get(probe, (None, None, False))
        data = list(csv.reader(open(path)))
        if len(data) < 3:
            continue
        h, u = data[0], data[1]
        ix = {k: h.index(k) for k in h}
        for r in data[2:]:
            kname = r[ix["Kernel Name"]].replace("void ", "").split("(")[0]
            if probe == "c3":  # 25 launches: keep one of each kernel
                pass
            dur = float(r[ix["gpu__time_duration.sum"]]) * time_scale(u[ix["gpu__time_duration.sum"]])
            dram = sum(float(r[ix[k]]) * unit_scale(u[ix[k]]) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            launch_rows = rows
            if probe == "c3" and "bwd" in kname:
                launch_rows = rows  # each block backward covers the whole batch
            alg = alg_bytes(kname, n, launch_rows, cplx) if n else None
            if probe == "c3" and "cascade_fwd" in kname:
                alg = 8 * n * rows  # x in, y out for the whole 12-block stack
            ach = alg / dur / 1e9 if alg else None
            g = lambda k: r[ix[k]] if k in ix else ""
            print(f"| {probe} | `{kname}` | {g('Grid Size')} x {g('Block Size')} | "
                  f"{g('launch__registers_per_thread')} | {dur * 1e6:.1f} us | {dram / 1e6:.1f} MB | "
                  + (f"{alg / 1e6:.1f} MB | {ach:.0f} | {ach / peak:.3f} | {dram / alg:.2f} |" if alg else "- | - | - | - |")
                  + f" {float(g('smsp__issue_active.avg.pct_of_peak_sustained_active') or 0):.1f} |"
                  f" {float(g('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active') or 0):.1f} |"
                  f" {g('smsp__sass_inst_executed_op_local_ld.sum')} |")


if __name__ == "__main__":
    main()
