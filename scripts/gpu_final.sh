#!/bin/bash
# Round-2 final evidence at HEAD: GPU suite, smoke, bench line (+ reference arm), configs, 2 ranks sharing the GPU,
# ncu launch list of bench.py, sanitizer suite.
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest.txt; cat $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; cat $O/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; cut -c1-200 $O/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; cut -c1-200 $O/bench_ref.json
timeout 900 python bench_configs.py --steps 20 > $O/configs.jsonl 2>$O/configs.err; cut -c1-160 $O/configs.jsonl
ACDC_SHARE_GPU=1 ACDC_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-dense > $O/bench_2rank_shared_gpu.json 2> $O/bench_2rank.err; cut -c1-200 $O/bench_2rank_shared_gpu.json
K='regex:acdc_|afdf_|cascade_|fft_rows'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$K" --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-dense > /dev/null 2>>$O/ncu.err
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_probe.py 2>&1 | grep -v "Host Frame\|^=========         " | head -c 20000 > $O/sanitize_$tool.txt
  echo "$tool: $(tail -1 $O/sanitize_$tool.txt)"
done
