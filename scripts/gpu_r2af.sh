#!/bin/bash
# Round-2 session U: C3 fused cascade forward CTA size (512 / 768 / 1024 threads) — A/B.
O=gpurun_out/r2af; mkdir -p $O
for rep in 1 2; do for v in c10b c10c768 c10c1024; do
  echo "{\"variant\": \"$v\", \"c3\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 300 python bench_configs.py --only c3 --steps 20 2>>$O/ab.err)}" >> $O/ab.jsonl
done; done
for v in c10b c10c768 c10c1024; do ACDC_LIB_PATH=gpurun_variants/$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:cascade_fwd -c 3 --log-file $O/ll_$v.csv python scripts/cascade_probe.py c3 > /dev/null 2>>$O/ncu.err; done
du -sh $O
