#!/bin/bash
# Round-2 session B: ncu (launch lists + one full capture per kernel family) and compute-sanitizer.
mkdir -p gpurun_out
T=r2b
K='regex:acdc_|afdf_|cascade_|fft_rows'
LL="--metrics gpu__time_duration.sum --clock-control none --csv"
FULL="--set full --import-source on --clock-control none"
run() { echo "== $*"; "$@" > /dev/null 2>>gpurun_out/${T}_ncu.err || echo "FAILED: $*"; }
# launch lists (cold-cache, serialised)
run timeout 300 ncu $LL -k "$K" --log-file gpurun_out/${T}_ll_m_cache.csv python scripts/size_probe.py 4096 16384 h2cache
run timeout 300 ncu $LL -k "$K" --log-file gpurun_out/${T}_ll_m_recompute.csv python scripts/size_probe.py 4096 16384 recompute
for n in 128 256 1024 8192 16384 32768; do
  run timeout 300 ncu $LL -k "$K" --log-file gpurun_out/${T}_ll_n$n.csv python scripts/size_probe.py $n 16384
done
run timeout 300 ncu $LL -k "$K" --log-file gpurun_out/${T}_ll_c3.csv python scripts/cascade_probe.py c3
run timeout 300 ncu $LL -k "$K" --log-file gpurun_out/${T}_ll_c5.csv python scripts/afdf_probe.py 8192 8192
# full captures: the last of the three probe iterations (skip the first two: warm tables / L2 state)
run timeout 600 ncu $FULL -k "$K" -s 6 -c 3 -o gpurun_out/${T}_full_m_cache python scripts/size_probe.py 4096 16384 h2cache
run timeout 600 ncu $FULL -k "$K" -s 6 -c 3 -o gpurun_out/${T}_full_m_recompute python scripts/size_probe.py 4096 16384 recompute
run timeout 600 ncu $FULL -k "$K" -s 8 -c 4 -o gpurun_out/${T}_full_n128 python scripts/size_probe.py 128 16384
run timeout 600 ncu $FULL -k "$K" -s 6 -c 3 -o gpurun_out/${T}_full_n8192 python scripts/size_probe.py 8192 16384
run timeout 600 ncu $FULL -k "$K" -s 6 -c 3 -o gpurun_out/${T}_full_n16384 python scripts/size_probe.py 16384 16384
run timeout 900 ncu $FULL -k "$K" -s 6 -c 3 -o gpurun_out/${T}_full_n32768 python scripts/size_probe.py 32768 4096
run timeout 900 ncu $FULL -k "$K" -s 25 -c 25 -o gpurun_out/${T}_full_c3 python scripts/cascade_probe.py c3
run timeout 600 ncu $FULL -k "$K" -s 4 -c 2 -o gpurun_out/${T}_full_c5 python scripts/afdf_probe.py 8192 8192
# race / sync / memory evidence
for tool in memcheck racecheck synccheck initcheck; do
  echo "== sanitizer $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_probe.py > gpurun_out/${T}_sanitize_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/${T}_sanitize_$tool.txt
  tail -4 gpurun_out/${T}_sanitize_$tool.txt
done
ls -la gpurun_out/ | grep $T
