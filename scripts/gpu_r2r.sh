#!/bin/bash
# Round-2 session R: compute-sanitizer at HEAD (half-length plan from N=2048, two-block cascade backward,
# deferred multi-block reduction), all four tools.
O=gpurun_out/r2r; mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_probe.py > $O/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -c 'Error' $O/sanitize_$tool.txt) error lines; $(tail -1 $O/sanitize_$tool.txt)"
done
