#!/bin/bash
# Round-2 session M: group-major unit mapping + spread grid (A/B with ACDC_GRID_SPREAD=0), GPU suite.
O=gpurun_out/r2m; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $O/pytest.txt; cat $O/pytest.txt
S="256:128 256:1024 128:16384 256:16384 512:16384 1024:16384 2048:16384 4096:16384 8192:16384 1024:512 4096:256"
for rep in 1 2; do for sp in 1 0; do
  ACDC_GRID_SPREAD=$sp timeout 300 python scripts/step_probe.py $S >> $O/spread.jsonl 2>>$O/err.txt
done; done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/r2m/spread.jsonl"):
    r = json.loads(l); d[(r["n"], r["rows"], r["spread"])].append(r["step_us"])
for (n, rows, sp), v in sorted(d.items()):
    print(n, rows, "spread" if sp == "1" else "packed", " ".join(f"{u:8.2f}" for u in v))
PY
