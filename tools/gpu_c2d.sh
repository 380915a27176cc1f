#!/bin/bash
O=gpurun_out/c2d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "T2 or C1 or C2 or slab" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for C in C3 C2; do timeout 600 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/bench_${C}.json 2>&1; done
MG_UNFUSED_COARSE=1 timeout 600 python bench.py --config C3 --no-cpu --no-e2e --steps 5 > $O/bench_C3_unfused.json 2>&1
