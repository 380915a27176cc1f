#!/bin/bash
O=gpurun_out/h8c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q -k "T3 or C4 or C5" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for C in C4 C5; do timeout 600 python bench.py --config $C --no-cpu --no-e2e --steps 3 > $O/bench_$C.json 2>&1; done
MG_UNFUSED_COARSE=1 timeout 600 python bench.py --config C5 --no-cpu --no-e2e --steps 3 > $O/bench_C5_unfused.json 2>&1
