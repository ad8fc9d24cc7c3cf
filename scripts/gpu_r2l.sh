#!/bin/bash
# Round-2 session L: two-block cascade backward restricted to N <= 2048; full GPU suite; C3/C4.
O=gpurun_out/r2l; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $O/pytest.txt; cat $O/pytest.txt
timeout 300 python bench_configs.py --only c3,c4 --steps 20 > $O/configs.jsonl 2>$O/configs.err; cut -c1-250 $O/configs.jsonl
