#!/bin/bash
# Round-2 session U: 2 ranks sharing the GPU through bench.py --gpus 2 (gloo) at HEAD; launch lists at N=128/256/512.
O=gpurun_out/r2ac; mkdir -p $O
ACDC_SHARE_GPU=1 ACDC_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-dense > $O/bench_2rank_shared_gpu.json 2> $O/bench_2rank.err; cut -c1-300 $O/bench_2rank_shared_gpu.json; tail -3 $O/bench_2rank.err
K='regex:acdc_|afdf_|cascade_|fft_rows'
for n in 128 256 512; do
  timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread --clock-control none --csv -k "$K" --log-file $O/ll_n$n.csv python scripts/size_probe.py $n 16384 > /dev/null 2>>$O/ncu.err
done
du -sh $O
