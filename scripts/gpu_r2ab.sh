#!/bin/bash
# Round-2 session U: fused-step epilogue with role-0 x prefetch + a stash (A/B vs the split kernel), tests, C1.
O=gpurun_out/r2ab; mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py -q 2>&1 | tail -4 > $O/pytest_step.txt; tail -2 $O/pytest_step.txt
for rep in 1 2 3; do for v in split xpre; do for r in 2 128; do
  echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py 256 $r 2>>$O/ab.err)}" >> $O/step_ab.jsonl
done; done; done

for v in split xpre; do ACDC_LIB_PATH=gpurun_variants/$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:acdc_step -c 5 --log-file $O/step_launches_$v.csv python scripts/c1_probe.py 256 128 > /dev/null 2>>$O/ncu.err; done
du -sh $O
