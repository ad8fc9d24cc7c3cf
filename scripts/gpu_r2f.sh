#!/bin/bash
# Round-2 session F: HL dy staging + split tables; A/B of HL variants; synccheck hypothesis for the HL kernels.
O=gpurun_out/r2f; mkdir -p $O
timeout 900 python -m pytest tests/test_hl_gpu.py tests/test_parity_gpu.py tests/test_fullshape_gpu.py -m gpu -q -x 2>&1 | tail -5 > $O/pytest.txt; cat $O/pytest.txt
timeout 600 python bench_configs.py --only sweep --steps 20 > $O/sweep.jsonl 2>$O/sweep.err; cut -c1-200 $O/sweep.jsonl
timeout 600 python scripts/ab_bench.py --n 16384 --trials 4 paper_1511_05946_b200/libacdc_b200.so gpurun_variants/hl_nbuf2.so > $O/ab_16384.txt 2>&1; tail -8 $O/ab_16384.txt
for n in 8192 16384 32768; do
  timeout 300 compute-sanitizer --tool synccheck python scripts/synccheck_hl.py $n 2>&1 | grep -v "Host Frame" | head -c 3000 > $O/sync_main_$n.txt; echo "main $n: $(tail -1 $O/sync_main_$n.txt)"
done
ACDC_LIB_PATH=gpurun_variants/hl_slotdyn.so timeout 300 compute-sanitizer --tool synccheck python scripts/synccheck_hl.py 16384 2>&1 | grep -v "Host Frame" | head -c 3000 > $O/sync_slotdyn.txt; echo "slotdyn: $(tail -1 $O/sync_slotdyn.txt)"
timeout 300 compute-sanitizer --tool racecheck python scripts/synccheck_hl.py 8192 2>&1 | tail -2 > $O/race_8192.txt; cat $O/race_8192.txt
