#!/bin/bash
# Round-2 session U: fused step — tests, CTA-size A/B (variants), ncu of the step kernel; K6 ncu comparison
# (selected metrics only: a --set full capture of the cuBLAS GEMMs exceeds gpurun's 64 MiB return limit).
O=gpurun_out/r2w; mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py -q 2>&1 | tail -4 > $O/pytest_step.txt; tail -2 $O/pytest_step.txt
for rep in 1 2; do for v in step128 step256 step512; do for r in 128 1024; do
  echo "{\"variant\": \"$v\", \"probe\": $(ACDC_LIB_PATH=gpurun_variants/$v.so timeout 120 python scripts/c1_probe.py 256 $r 2>>$O/ab.err)}" >> $O/step_cta_ab.jsonl
done; done; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:acdc_step -c 1 -o $O/step_full python scripts/c1_probe.py 256 128 > /dev/null 2>>$O/ncu.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:acdc_ -c 60 --log-file $O/c1_launches.csv python scripts/c1_probe.py 256 128 > /dev/null 2>>$O/ncu.err
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size
K6_NCU=1 timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/k6_metrics.csv python scripts/k6_probe.py > $O/k6_ncu_stdout.txt 2>>$O/ncu.err
timeout 300 python scripts/k6_probe.py > $O/k6_probe.json 2>>$O/k6.err
du -sh $O; ls -la $O
