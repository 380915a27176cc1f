#!/bin/bash
O=gpurun_out/gf; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C3 C5 C4 C2; do timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}.json 2>&1; done
