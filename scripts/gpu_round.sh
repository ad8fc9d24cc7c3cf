#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list, ncu full capture of the hot kernels.
# usage: scripts/gpu_round.sh [tag] [tests=1] [full=1]
TAG=${1:-r}
TESTS=${2:-1}
FULL=${3:-1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${TAG}_smi.txt
if [ "$TESTS" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/${TAG}_pytest.txt
  cat gpurun_out/${TAG}_pytest.txt
fi
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 5 --warmup 3 --mode h2cache --no-cpu-baseline --no-e2e --no-dense > /dev/null 2>&1
if [ "$FULL" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:acdc_ -s 8 -c 4 -o gpurun_out/${TAG}_prof \
    python bench.py --steps 3 --warmup 3 --mode h2cache --no-cpu-baseline --no-e2e --no-dense > gpurun_out/${TAG}_ncu.log 2>&1
  tail -2 gpurun_out/${TAG}_ncu.log
fi
