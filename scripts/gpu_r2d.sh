#!/bin/bash
# Round-2 session D: full GPU suite, sweep (HL A/B), K6 probe + ncu of its two kernels.
O=gpurun_out/r2d; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/pytest.txt; cat $O/pytest.txt
timeout 600 python bench_configs.py --only sweep --steps 20 > $O/sweep.jsonl 2>$O/sweep.err
timeout 300 python scripts/k6_probe.py > $O/k6.json 2>$O/k6.err; cat $O/k6.json; tail -3 $O/k6.err
timeout 600 ncu --set full --clock-control none -k 'regex:fft_rows|gemm|nvjet|sm100|cutlass|Kernel' -c 6 -o /tmp/k6 python scripts/k6_probe.py > /dev/null 2>>$O/ncu.err
ncu -i /tmp/k6.ncu-rep --page raw --csv > $O/k6_raw.csv 2>>$O/ncu.err
python scripts/summarize_ncu.py /tmp/k6.ncu-rep $O --name sum_k6 --traffic $O/traffic_k6.json > /dev/null 2>>$O/ncu.err
du -sh $O
