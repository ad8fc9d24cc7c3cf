#!/bin/bash
# Round-2 session U (re-entry): evidence at HEAD — GPU suite, smoke, bench line, reference arm, configs, launch list.
O=gpurun_out/r2u; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/pytest.txt; tail -3 $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; cut -c1-300 $O/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; cut -c1-200 $O/bench_ref.json
timeout 900 python bench_configs.py --steps 20 > $O/configs.jsonl 2>$O/configs.err; cut -c1-200 $O/configs.jsonl
K='regex:acdc_|afdf_|cascade_|fft_rows'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$K" --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-dense > /dev/null 2>>$O/ncu.err
wc -l $O/launches.csv
