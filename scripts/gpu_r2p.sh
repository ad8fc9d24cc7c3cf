#!/bin/bash
# Round-2 session P: evidence at HEAD (GPU suite, bench line, configs).
O=gpurun_out/r2p; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $O/pytest.txt; cat $O/pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; cut -c1-300 $O/bench.json
timeout 900 python bench_configs.py --steps 20 > $O/configs.jsonl 2>$O/configs.err; cut -c1-220 $O/configs.jsonl
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; cut -c1-300 $O/bench_ref.json
