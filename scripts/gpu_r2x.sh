#!/bin/bash
# Round-2 session U: fused step with the first pair's loads ahead of the table staging (A/B variants), tests.
O=gpurun_out/r2x; mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py -q 2>&1 | tail -4 > $O/pytest_step.txt; tail -2 $O/pytest_step.txt
for rep in 1 2 3; do for v in nopre256 pre256 pre128; do for r in 2 128; do
  echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py 256 $r 2>>$O/ab.err)}" >> $O/step_ab.jsonl
done; done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:acdc_step --log-file $O/step_launches.csv python scripts/c1_probe.py 256 128 > /dev/null 2>>$O/ncu.err
for v in nopre256 pre256 pre128; do ACDC_LIB_PATH=gpurun_variants/$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:acdc_step -c 5 --log-file $O/step_launches_$v.csv python scripts/c1_probe.py 256 128 > /dev/null 2>>$O/ncu.err; done
du -sh $O
