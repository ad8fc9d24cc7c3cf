"""Summarise an ncu --set full report (and optional launch-list CSV) into profiles/.

usage: python scripts/summarize_ncu.py <prof.ncu-rep> <out_dir> [launches.csv] [--name NAME] [--traffic PATH]

Writes <out_dir>/ncu_summary.md (per-kernel key metrics, instruction mix) and
updates profiles/traffic.json (dram read+write bytes per launch, per kernel)
which bench.py reports as roofline.traffic.
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import Counter

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % of peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__sass_inst_executed_op_local_ld.sum", "local (spill) loads"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall lg_throttle"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def short(name):
    return name.split("(")[0].replace("void ", "").strip()


def main():
    argv = list(sys.argv[1:])
    opts = {}
    for key in ("--name", "--traffic"):
        if key in argv:
            i = argv.index(key)
            opts[key] = argv[i + 1]
            del argv[i:i + 2]
    rep, out_dir = argv[0], argv[1]
    launches = argv[2] if len(argv) > 2 else None
    os.makedirs(out_dir, exist_ok=True)
    rows = ncu_csv(["-i", rep, "--page", "raw"])
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu summary: `{os.path.basename(rep)}`", ""]
    traffic = {}
    for r in rows[2:]:
        kname = r[hdr.index("Kernel Name")]
        lines.append(f"## {kname}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        vals = {}
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                vals[k] = r[i]
                lines.append(f"| {label} (`{k}`) | {r[i]} | {units[i]} |")
        try:
            rd = float(vals["dram__bytes_read.sum"]) * (1e6 if "M" in units[hdr.index("dram__bytes_read.sum")] else 1)
            wr_u = units[hdr.index("dram__bytes_write.sum")]
            wr = float(vals["dram__bytes_write.sum"]) * (1e9 if wr_u.startswith("G") else 1e6 if wr_u.startswith("M") else 1)
            rd_u = units[hdr.index("dram__bytes_read.sum")]
            rd = float(vals["dram__bytes_read.sum"]) * (1e9 if rd_u.startswith("G") else 1e6 if rd_u.startswith("M") else 1)
            key = short(kname).split("<")[0].split("::")[-1]
            traffic.setdefault(key, rd + wr)
        except Exception:
            pass
        lines.append("")
    # instruction mix from the source page
    for kern in sorted({short(r[hdr.index("Kernel Name")]).split("<")[0].split("::")[-1] for r in rows[2:]}):
        src = ncu_csv(["-i", rep, "--page", "source", "--kernel-name", f"regex:{kern}"])
        if len(src) < 3:
            continue
        h = src[1]
        try:
            ie = h.index("Instructions Executed")
        except ValueError:
            continue
        c = Counter()
        tot = 0
        for r in src[2:]:
            if len(r) <= ie or not r[ie].isdigit():
                continue
            toks = r[1].strip().split()
            if not toks:
                continue
            op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
            c[op] += int(r[ie])
            tot += int(r[ie])
        if tot:
            lines.append(f"### instruction mix: {kern}")
            lines.append("")
            lines.append("| opcode | share |")
            lines.append("|---|---|")
            for op, v in c.most_common(12):
                lines.append(f"| {op} | {100 * v / tot:.1f}% |")
            lines.append("")
    if launches and os.path.exists(launches):
        lr = list(csv.reader(open(launches)))
        try:
            hi = next(i for i, r in enumerate(lr) if "Kernel Name" in r)
            h = lr[hi]
            ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
            per = {}
            for r in lr[hi + 1:]:
                if len(r) > vi and r[mi] == "gpu__time_duration.sum":
                    per.setdefault(short(r[ki]), []).append(float(r[vi].replace(",", "")))
            total = sum(sum(v) for v in per.values())
            lines.append("## launch list (ncu, cold-cache, serialised)")
            lines.append("")
            lines.append("| kernel | launches | mean duration | share of listed time |")
            lines.append("|---|---|---|---|")
            for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
                lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / total:.1f}% |")
            lines.append("")
        except StopIteration:
            pass
    with open(os.path.join(out_dir, opts.get("--name", "ncu_summary") + ".md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tpath = opts.get("--traffic") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                                                  "traffic.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    old.update(traffic)
    with open(tpath, "w") as f:
        json.dump(old, f, indent=1)
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
