#!/bin/bash
# Round-2 session U: last validation at HEAD — GPU suite + smoke + bench line.
O=gpurun_out/r2ah; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest.txt; cat $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; cat $O/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; cut -c1-200 $O/bench.json
