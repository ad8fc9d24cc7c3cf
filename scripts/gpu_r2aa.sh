#!/bin/bash
# Round-2 session U: fused-step epilogue with overlapped loads (A/B vs the previous split kernel), tests, C1.
O=gpurun_out/r2aa; mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py -q 2>&1 | tail -4 > $O/pytest_step.txt; tail -2 $O/pytest_step.txt
for rep in 1 2 3; do for v in split fin; do for r in 2 128; do
  echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py 256 $r 2>>$O/ab.err)}" >> $O/step_ab.jsonl
done; done; done
timeout 300 python bench_configs.py --only c1 --steps 20 > $O/c1.jsonl 2>$O/c1.err; cut -c1-300 $O/c1.jsonl
for v in split fin; do ACDC_LIB_PATH=gpurun_variants/$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:acdc_step -c 5 --log-file $O/step_launches_$v.csv python scripts/c1_probe.py 256 128 > /dev/null 2>>$O/ncu.err; done
du -sh $O
