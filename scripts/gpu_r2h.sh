#!/bin/bash
# Round-2 session H (re-entry: HEAD measurement): full GPU suite, bench line, configs, ncu of the HL kernels at HEAD.
O=gpurun_out/r2h; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > $O/pytest.txt; tail -3 $O/pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; cat $O/bench.json | cut -c1-300
timeout 900 python bench_configs.py --steps 20 > $O/configs.jsonl 2>$O/configs.err; cut -c1-250 $O/configs.jsonl
K='regex:acdc_|afdf_|cascade_|fft_rows'
for spec in "n8192 6 3 8192 16384" "n16384 6 3 16384 16384" "n32768 6 3 32768 4096"; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$K" --log-file $O/ll_$1.csv python scripts/size_probe.py $4 $5 > /dev/null 2>>$O/ncu.err
  timeout 900 ncu --set full --import-source on --clock-control none -k "$K" -s $2 -c $3 -o /tmp/full_$1 python scripts/size_probe.py $4 $5 > /dev/null 2>>$O/ncu.err
  python scripts/summarize_ncu.py /tmp/full_$1.ncu-rep $O $O/ll_$1.csv --name sum_$1 --traffic $O/traffic_$1.json > /dev/null 2>>$O/ncu.err
  ncu -i /tmp/full_$1.ncu-rep --page raw --csv > $O/raw_$1.csv 2>/dev/null
done
du -sh $O
