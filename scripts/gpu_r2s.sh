#!/bin/bash
# Round-2 session S: sanitizer suite at HEAD (dummy mbarrier before TMEM allocation), TMEM probe, tests, bench.
O=gpurun_out/r2s; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 scripts/synccheck_tmem_probe.cu -o /tmp/sc_probe
for m in 0 1 2; do timeout 120 compute-sanitizer --tool synccheck /tmp/sc_probe $m 2>&1 | grep -v "Host Frame\|^=========         "; done > $O/synccheck_tmem_probe.txt 2>&1
grep "mode\|SUMMARY" $O/synccheck_tmem_probe.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_probe.py > $O/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(tail -1 $O/sanitize_$tool.txt)"
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $O/pytest.txt; cat $O/pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; cut -c1-250 $O/bench.json
