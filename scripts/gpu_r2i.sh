#!/bin/bash
# Round-2 session I: L2 cache-hint variants (A/B at N=4096), launch lists of C1 and C3 at HEAD.
O=gpurun_out/r2i; mkdir -p $O
timeout 900 python scripts/ab_bench.py --n 4096 --trials 6 gpurun_variants/base12.so gpurun_variants/h2keep12.so gpurun_variants/stcs12.so gpurun_variants/both12.so > $O/ab_l2.txt 2>&1; tail -5 $O/ab_l2.txt
K='regex:acdc_|afdf_|cascade_|fft_rows'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$K" --log-file $O/ll_c1.csv python scripts/size_probe.py 256 128 > /dev/null 2>>$O/ncu.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$K" --log-file $O/ll_c3.csv python scripts/cascade_probe.py c3 > /dev/null 2>>$O/ncu.err
python - <<'PY'
import csv, collections
for f in ("gpurun_out/r2i/ll_c1.csv", "gpurun_out/r2i/ll_c3.csv"):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")); v = v / 1000 if r[ui] == "nsecond" else v
        k = r[ki][:60]; agg.setdefault(k, []).append(v)
    print(f)
    for k, v in agg.items(): print(f"  {k:60s} n={len(v):3d} mean={sum(v)/len(v):8.2f} us")
PY
