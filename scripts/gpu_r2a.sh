#!/bin/bash
# Round-2 session A: GPU tests (incl. full-shape parity, DP), bench, multi-rank sanity, configs.
mkdir -p gpurun_out
T=r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${T}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=25 > gpurun_out/${T}_pytest.txt 2>&1
tail -40 gpurun_out/${T}_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
cat gpurun_out/${T}_bench.json; tail -3 gpurun_out/${T}_bench.err
ACDC_DIST_BACKEND=gloo ACDC_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-dense --no-e2e > gpurun_out/${T}_bench2.json 2> gpurun_out/${T}_bench2.err
cat gpurun_out/${T}_bench2.json; tail -3 gpurun_out/${T}_bench2.err
timeout 900 python bench_configs.py --steps 20 > gpurun_out/${T}_configs.jsonl 2> gpurun_out/${T}_configs.err
cat gpurun_out/${T}_configs.jsonl; tail -3 gpurun_out/${T}_configs.err
ACDC_DIST_BACKEND=gloo ACDC_SHARE_GPU=1 timeout 600 python bench_configs.py --only c4,c5 --gpus 2 --steps 10 --c5-rows 16384 > gpurun_out/${T}_configs2.jsonl 2> gpurun_out/${T}_configs2.err
cat gpurun_out/${T}_configs2.jsonl; tail -3 gpurun_out/${T}_configs2.err
