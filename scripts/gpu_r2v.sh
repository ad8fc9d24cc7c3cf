#!/bin/bash
# Round-2 session U: fused small-batch step (acdc_step_f32) — tests, C1 timing, probe, ncu of the step kernel.
O=gpurun_out/r2v; mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py -q -x 2>&1 | tail -15 > $O/pytest_step.txt; tail -3 $O/pytest_step.txt
timeout 300 python bench_configs.py --only c1 --steps 20 > $O/c1.jsonl 2>$O/c1.err; cat $O/c1.jsonl; tail -3 $O/c1.err
for r in 2 64 128 256; do timeout 120 python scripts/c1_probe.py 256 $r >> $O/c1_probe.jsonl 2>>$O/c1.err; done
for n in 512 1024 2048 4096; do timeout 120 python scripts/c1_probe.py $n 8 >> $O/c1_probe.jsonl 2>>$O/c1.err; done
cat $O/c1_probe.jsonl
timeout 300 ncu --set full --import-source on --clock-control none -k regex:acdc_ -c 6 -o $O/c1_full python scripts/c1_probe.py 256 128 > /dev/null 2>>$O/ncu.err
ls -la $O
