#!/bin/bash
# Round-2 session Q: ncu evidence for the metric shape on the half-length plan (N=4096): launch list of
# bench.py, full capture of the forward / backward / reduction, source page; bench line after.
O=gpurun_out/r2q; mkdir -p $O
K='regex:acdc_|afdf_|cascade_|fft_rows'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "$K" --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-dense > /dev/null 2>>$O/ncu.err
timeout 900 ncu --set full --import-source on --clock-control none -k "$K" -s 3 -c 3 -o /tmp/full_m python scripts/size_probe.py 4096 16384 > /dev/null 2>>$O/ncu.err
python scripts/summarize_ncu.py /tmp/full_m.ncu-rep $O $O/launches.csv --name sum_m_hl --traffic $O/traffic.json > /dev/null 2>>$O/ncu.err
ncu -i /tmp/full_m.ncu-rep --page raw --csv > $O/raw_m_hl.csv 2>/dev/null
ncu -i /tmp/full_m.ncu-rep --page source --csv > $O/src_m_hl.csv 2>/dev/null
cat $O/traffic.json
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; cut -c1-400 $O/bench.json
