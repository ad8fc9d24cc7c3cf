#!/bin/bash
# Round-2 session J: deferred cascade reductions (tests + C3), h2 normal-cached default, C1 breakdown + ncu.
O=gpurun_out/r2j; mkdir -p $O
timeout 900 python -m pytest tests/test_cascade_gpu.py tests/test_parity_gpu.py tests/test_dp_gpu.py -m gpu -q -x 2>&1 | tail -5 > $O/pytest.txt; cat $O/pytest.txt
timeout 300 python bench_configs.py --only c1,c3 --steps 20 > $O/configs.jsonl 2>$O/configs.err; cut -c1-300 $O/configs.jsonl
for r in 128 1024; do timeout 120 python scripts/c1_probe.py 256 $r; done | tee $O/c1_probe.jsonl
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; cut -c1-200 $O/bench.json
K='regex:acdc_|afdf_|cascade_|fft_rows'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$K" --log-file $O/ll_c3.csv python scripts/cascade_probe.py c3 > /dev/null 2>>$O/ncu.err
timeout 600 ncu --set full --import-source on --clock-control none -k "$K" -s 3 -c 3 -o /tmp/full_c1 python scripts/size_probe.py 256 128 > /dev/null 2>>$O/ncu.err
python scripts/summarize_ncu.py /tmp/full_c1.ncu-rep $O --name sum_c1 > /dev/null 2>>$O/ncu.err
ncu -i /tmp/full_c1.ncu-rep --page raw --csv > $O/raw_c1.csv 2>/dev/null
ncu -i /tmp/full_c1.ncu-rep --page source --csv > $O/src_c1.csv 2>/dev/null
