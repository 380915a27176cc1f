#!/bin/bash
O=gpurun_out/h8b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "T3 or C4 or C5" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for M in 1 2; do for C in C4 C5; do MG_H8_MINB=$M timeout 600 python bench.py --config $C --no-cpu --no-e2e --steps 3 > $O/bench_${C}_$M.json 2>&1; done; done
