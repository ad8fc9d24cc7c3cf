#!/bin/bash
# Round-2 session U: split-role step at 128-thread CTAs in a 16-CTA (non-portable) cluster vs 256 x 8 — A/B, C1.
O=gpurun_out/r2ag; mkdir -p $O
for rep in 1 2 3; do for v in s256c8 s128c16; do for r in 2 128; do
  echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py 256 $r 2>>$O/ab.err)}" >> $O/ab.jsonl
done; done; done
ACDC_LIB_PATH=gpurun_variants/s128c16.so timeout 300 python -m pytest tests/test_step_gpu.py -q -k "256" 2>&1 | tail -2 > $O/pytest_s128c16.txt
for v in s256c8 s128c16; do ACDC_LIB_PATH=gpurun_variants/$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:acdc_step -c 5 --log-file $O/ll_$v.csv python scripts/c1_probe.py 256 128 > /dev/null 2>>$O/ncu.err; done
du -sh $O
