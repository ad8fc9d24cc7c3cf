#!/bin/bash
# Round-2 session O: shared-memory carveout preference sweep (driver default vs min vs 50%).
O=gpurun_out/r2o; mkdir -p $O
S="128:16384 256:16384 512:16384 1024:16384 2048:16384 4096:16384 8192:16384 16384:16384 32768:4096"
for rep in 1 2; do
for co in -1 0 50; do
  if [ "$co" = "-1" ]; then unset ACDC_CARVEOUT; else export ACDC_CARVEOUT=$co; fi
  timeout 300 python scripts/step_probe.py $S | sed "s/^{/{\"carveout\": $co, /" >> $O/sweep.jsonl
  timeout 300 python bench_configs.py --only c3,c4,c5 --steps 10 | sed "s/^{/{\"carveout\": $co, /" >> $O/configs.jsonl 2>>$O/err.txt
done; done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/r2o/sweep.jsonl"):
    r = json.loads(l); d[(r["n"], r["carveout"])].append(r["step_us"])
for (n, co), v in sorted(d.items()):
    print("sweep", n, co, " ".join(f"{u:9.2f}" for u in v))
d = collections.defaultdict(list)
for l in open("gpurun_out/r2o/configs.jsonl"):
    r = json.loads(l); k = r["config"][:3]; d[(k, r["carveout"])].append(r.get("fused_ms", r.get("ms_per_step")))
for (k, co), v in sorted(d.items()):
    print("config", k, co, " ".join(f"{u:9.4f}" for u in v))
PY
