#!/bin/bash
# Round-2 final evidence (session U, after the small-N forward CTAs) at HEAD: GPU suite, smoke, bench line (+ reference arm), configs,
# ncu launch list of bench.py, ncu of the fused step kernel, sanitizer suite.
O=gpurun_out/final4; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest.txt; cat $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; cat $O/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; cut -c1-200 $O/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; cut -c1-200 $O/bench_ref.json
timeout 900 python bench_configs.py --steps 20 > $O/configs.jsonl 2>$O/configs.err; cut -c1-200 $O/configs.jsonl
K='regex:acdc_|afdf_|cascade_|fft_rows'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$K" --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-dense > /dev/null 2>>$O/ncu.err
timeout 300 ncu --set full --import-source on --clock-control none -k regex:acdc_step -c 1 -o /tmp/step_full python scripts/c1_probe.py 256 128 > /dev/null 2>>$O/ncu.err
python scripts/summarize_ncu.py /tmp/step_full.ncu-rep $O --name sum_step > /dev/null 2>>$O/ncu.err; ls $O
du -sh $O
