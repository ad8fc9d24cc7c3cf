#!/bin/bash
# Round-2 session U: split-role fused step (two groups per row pair) — tests, A/B vs the single-role kernel, C1.
O=gpurun_out/r2z; mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py -q 2>&1 | tail -4 > $O/pytest_step.txt; tail -2 $O/pytest_step.txt
for rep in 1 2 3; do for v in nosplit split; do for r in 2 128; do
  echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py 256 $r 2>>$O/ab.err)}" >> $O/step_ab.jsonl
done; done; done
for n in 512; do for v in nosplit split; do echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py $n 64 2>>$O/ab.err)}" >> $O/step_ab.jsonl; done; done
timeout 300 python bench_configs.py --only c1 --steps 20 > $O/c1.jsonl 2>$O/c1.err; cut -c1-300 $O/c1.jsonl
timeout 300 ncu --set full --import-source on --clock-control none -k regex:acdc_step -c 1 -o /tmp/step_full python scripts/c1_probe.py 256 128 > /dev/null 2>>$O/ncu.err
python scripts/summarize_ncu.py /tmp/step_full.ncu-rep $O --name sum_step2 > /dev/null 2>>$O/ncu.err
du -sh $O
