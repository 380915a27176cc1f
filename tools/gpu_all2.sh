#!/bin/bash
# full GPU suite + bench of all configs
O=gpurun_out/$1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C1 C2 C3 C4 C5; do
timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}.json 2>&1
done
