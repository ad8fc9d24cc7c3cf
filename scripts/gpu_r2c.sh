#!/bin/bash
# Round-2 session C: HL tests, ncu summaries produced ON the box (reports are too big to ship back), sanitizers.
mkdir -p gpurun_out/r2c
O=gpurun_out/r2c
timeout 900 python -m pytest tests/test_hl_gpu.py tests/test_parity_gpu.py tests/test_cascade_gpu.py tests/test_sgd_fused_gpu.py -m gpu -q -x 2>&1 | tail -15 > $O/pytest_hl.txt
cat $O/pytest_hl.txt
timeout 600 python bench_configs.py --only sweep --steps 20 > $O/sweep.jsonl 2>$O/sweep.err; cat $O/sweep.jsonl | cut -c1-200
ACDC_HL=0 timeout 600 python bench_configs.py --only sweep --steps 20 > $O/sweep_hl0.jsonl 2>>$O/sweep.err
K='regex:acdc_|afdf_|cascade_|fft_rows'
LL="--metrics gpu__time_duration.sum --clock-control none --csv"
FULL="--set full --import-source on --clock-control none"
cap() {  # name skip count probe...
  local name=$1 skip=$2 cnt=$3; shift 3
  timeout 300 ncu $LL -k "$K" --log-file $O/ll_$name.csv "$@" > /dev/null 2>>$O/ncu.err
  timeout 900 ncu $FULL -k "$K" -s $skip -c $cnt -o /tmp/full_$name "$@" > /dev/null 2>>$O/ncu.err
  python scripts/summarize_ncu.py /tmp/full_$name.ncu-rep $O $O/ll_$name.csv --name sum_$name --traffic $O/traffic_$name.json > /dev/null 2>>$O/ncu.err
  ncu -i /tmp/full_$name.ncu-rep --page raw --csv > $O/raw_$name.csv 2>/dev/null
  echo "captured $name: $(ls -la $O/sum_$name.md 2>/dev/null | awk '{print $5}') bytes"
}
cap m_cache 6 3 python scripts/size_probe.py 4096 16384 h2cache
cap m_recompute 6 3 python scripts/size_probe.py 4096 16384 recompute
cap n128 8 4 python scripts/size_probe.py 128 16384
cap n8192 6 3 python scripts/size_probe.py 8192 16384
cap n16384 6 3 python scripts/size_probe.py 16384 16384
cap n32768 6 3 python scripts/size_probe.py 32768 4096
cap c3 25 25 python scripts/cascade_probe.py c3
cap c5 4 2 python scripts/afdf_probe.py 8192 8192
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 30 python scripts/sanitize_probe.py 2>&1 | head -c 60000 > $O/sanitize_$tool.txt
  echo "== $tool: $(tail -2 $O/sanitize_$tool.txt | tr '\n' ' ')"
done
du -sh $O
