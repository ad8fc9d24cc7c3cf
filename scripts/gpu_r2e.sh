#!/bin/bash
# Round-2 session E: GPU suite, configs (C3 gather path, graphed sweep), K6 GEMM ncu, sanitizers after the race fix.
O=gpurun_out/r2e; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/pytest.txt; cat $O/pytest.txt
timeout 900 python bench_configs.py --only c1,c3,sweep,c5 --steps 20 > $O/configs.jsonl 2>$O/configs.err; cut -c1-220 $O/configs.jsonl; tail -2 $O/configs.err
K6_NCU=1 timeout 600 ncu --set full --clock-control none -c 12 -o /tmp/k6g python scripts/k6_probe.py > /dev/null 2>>$O/ncu.err
ncu -i /tmp/k6g.ncu-rep --page raw --csv > $O/k6g_raw.csv 2>>$O/ncu.err
python scripts/summarize_ncu.py /tmp/k6g.ncu-rep $O --name sum_k6g --traffic $O/traffic_k6g.json > /dev/null 2>>$O/ncu.err
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 30 python scripts/sanitize_probe.py 2>&1 | head -c 60000 > $O/sanitize_$tool.txt
  echo "== $tool: $(tail -2 $O/sanitize_$tool.txt | tr '\n' ' ')"
done
du -sh $O
