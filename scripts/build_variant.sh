#!/bin/bash
# Build an experimental variant of libacdc_b200.so (single size, extra -D flags).
# usage: scripts/build_variant.sh NAME LOGN "-DFLAG=1 ..."
set -e
NAME=$1; LOGN=$2; FLAGS=$3
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/variants
mkdir -p $OUT/$NAME
for f in $ROOT/paper_1511_05946_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -DACDC_ONLY_LOGN=$LOGN $FLAGS -I $ROOT/include -c $f -o $OUT/$NAME/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $OUT/$NAME/*.o -o $ROOT/gpurun_variants/$NAME.so 2>/dev/null || {
  mkdir -p $ROOT/gpurun_variants
  nvcc -gencode arch=compute_100a,code=sm_100a -shared $OUT/$NAME/*.o -o $ROOT/gpurun_variants/$NAME.so
}
echo $ROOT/gpurun_variants/$NAME.so
