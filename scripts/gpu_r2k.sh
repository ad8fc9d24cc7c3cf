#!/bin/bash
# Round-2 session K: two-block fused cascade backward (tests, C3/C4 A/B against one block per launch).
O=gpurun_out/r2k; mkdir -p $O
timeout 900 python -m pytest tests/test_cascade_gpu.py tests/test_fullshape_gpu.py tests/test_dp_gpu.py tests/test_sgd_fused_gpu.py -m gpu -q -x 2>&1 | tail -5 > $O/pytest.txt; cat $O/pytest.txt
for rep in 1 2; do
for pair in 1 0; do
  ACDC_CASCADE_PAIR=$pair timeout 300 python bench_configs.py --only c3,c4 --steps 20 > $O/configs_pair$pair.$rep.jsonl 2>$O/configs.err
  echo "pair=$pair rep=$rep"; cut -c1-220 $O/configs_pair$pair.$rep.jsonl
done
done
K='regex:acdc_|afdf_|cascade_|fft_rows'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$K" --log-file $O/ll_c3.csv python scripts/cascade_probe.py c3 > /dev/null 2>>$O/ncu.err
