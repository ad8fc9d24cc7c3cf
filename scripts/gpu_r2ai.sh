#!/bin/bash
# Round-2 session U: half-length forward at 1024-thread CTAs for N = 1024 / 2048 (batch 16384) — A/B.
O=gpurun_out/r2ai; mkdir -p $O
for rep in 1 2 3; do
  for v in h10b h10f1024; do echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py 1024 16384 2>>$O/ab.err)}" >> $O/ab.jsonl; done
  for v in h11b h11f1024; do echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py 2048 16384 2>>$O/ab.err)}" >> $O/ab.jsonl; done
done
du -sh $O
