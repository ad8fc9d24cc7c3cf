#!/bin/bash
# Round-2 session N: shared-memory carveout experiment (C1 latency), fwd latency at 2 rows.
O=gpurun_out/r2n; mkdir -p $O
for co in -1 100 50 0; do
  if [ "$co" = "-1" ]; then unset ACDC_CARVEOUT; else export ACDC_CARVEOUT=$co; fi
  echo "carveout=$co"
  timeout 120 python scripts/c1_probe.py 256 128
  timeout 120 python scripts/c1_probe.py 256 2
  timeout 120 python scripts/c1_probe.py 4096 256
  timeout 200 python scripts/step_probe.py 4096:16384 1024:16384
done 2>&1 | tee $O/carveout.txt
