#!/bin/bash
# Round-2 session U: N=256 at batch 16384 with 1024-thread CTAs (all 8192 row pairs in one wave) — A/B.
O=gpurun_out/r2ad; mkdir -p $O
for rep in 1 2 3; do for v in c8base c8f1024 c8fb1024; do
  echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py 256 16384 2>>$O/ab.err)}" >> $O/ab.jsonl
done; done
for v in c8base c8fb1024; do ACDC_LIB_PATH=gpurun_variants/$v.so timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv -k regex:acdc_ -c 9 --log-file $O/ll_$v.csv python scripts/c1_probe.py 256 16384 > /dev/null 2>>$O/ncu.err; done
du -sh $O
