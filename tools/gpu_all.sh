#!/bin/bash
# full GPU test suite + bench of all configs (no cpu/e2e). usage: bash tools/gpu_all.sh <tag>
O=gpurun_out/$1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for C in C1 C2 C3 C4 C5; do timeout 600 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/bench_$C.json 2>&1; done
