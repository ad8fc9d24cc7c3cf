#!/bin/bash
# Round-2 session U: ncu --set full of the metric-shape kernels at HEAD (summary, traffic), launch lists at N=8192/16384.
O=gpurun_out/r2y; mkdir -p $O
K='regex:acdc_|afdf_|cascade_|fft_rows'
cap() {  # name skip count probe...
  local name=$1 skip=$2 cnt=$3; shift 3
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$K" --log-file $O/ll_$name.csv "$@" > /dev/null 2>>$O/ncu.err
  timeout 900 ncu --set full --import-source on --clock-control none -k "$K" -s $skip -c $cnt -o /tmp/full_$name "$@" > /dev/null 2>>$O/ncu.err
  python scripts/summarize_ncu.py /tmp/full_$name.ncu-rep $O $O/ll_$name.csv --name sum_$name --traffic $O/traffic_$name.json > /dev/null 2>>$O/ncu.err
  echo "captured $name: $(ls -la $O/sum_$name.md 2>/dev/null | awk '{print $5}') bytes"
}
cap m_hl 6 3 python scripts/size_probe.py 4096 16384 h2cache
cap n8192 6 3 python scripts/size_probe.py 8192 16384
cap n16384 6 3 python scripts/size_probe.py 16384 16384
du -sh $O
