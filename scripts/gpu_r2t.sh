#!/bin/bash
# Round-2 session T: ncu captures of every shipped kernel at HEAD (summaries + raw CSV for the roofline table).
O=gpurun_out/r2t; mkdir -p $O
K='regex:acdc_|afdf_|cascade_|fft_rows'
LL="--metrics gpu__time_duration.sum --clock-control none --csv"
FULL="--set full --import-source on --clock-control none"
cap() {  # name skip count probe...
  local name=$1 skip=$2 cnt=$3; shift 3
  timeout 300 ncu $LL -k "$K" --log-file $O/ll_$name.csv "$@" > /dev/null 2>>$O/ncu.err
  timeout 900 ncu $FULL -k "$K" -s $skip -c $cnt -o /tmp/full_$name "$@" > /dev/null 2>>$O/ncu.err
  python scripts/summarize_ncu.py /tmp/full_$name.ncu-rep $O $O/ll_$name.csv --name sum_$name --traffic $O/traffic_$name.json > /dev/null 2>>$O/ncu.err
  ncu -i /tmp/full_$name.ncu-rep --page raw --csv > $O/raw_$name.csv 2>/dev/null
  echo "captured $name: $(ls -la $O/sum_$name.md 2>/dev/null | awk '{print $5}') bytes"
}
cap m_cache 6 3 python scripts/size_probe.py 4096 16384 h2cache
cap m_recompute 6 3 python scripts/size_probe.py 4096 16384 recompute
cap n128 8 4 python scripts/size_probe.py 128 16384
cap n256 6 3 python scripts/size_probe.py 256 16384
cap n1024 6 3 python scripts/size_probe.py 1024 16384
cap n2048 6 3 python scripts/size_probe.py 2048 16384
cap n8192 6 3 python scripts/size_probe.py 8192 16384
cap n16384 6 3 python scripts/size_probe.py 16384 16384
cap n32768 6 3 python scripts/size_probe.py 32768 4096
cap c3 8 8 python scripts/cascade_probe.py c3
cap c5 4 2 python scripts/afdf_probe.py 8192 8192
python scripts/roofline_table.py $O > $O/roofline_head.md; wc -l $O/roofline_head.md
du -sh $O
