#!/bin/bash
# Round-2 session U: N=256 forward on 1024-thread CTAs — GPU suite; N=512 A/B (768 vs 1024 forward CTAs).
O=gpurun_out/r2ae; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest.txt; cat $O/pytest.txt
for rep in 1 2 3; do for v in c9base c9f1024; do
  echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py 512 16384 2>>$O/ab.err)}" >> $O/ab.jsonl
done; echo "{\"variant\": \"main\", \"probe\": $(timeout 120 python scripts/c1_probe.py 256 16384 2>>$O/ab.err)}" >> $O/ab.jsonl; done
du -sh $O
