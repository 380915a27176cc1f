#!/bin/bash
O=gpurun_out/c5da; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
for m in 1 0; do MG_DENSE_ROWS=$m timeout 300 python bench.py --config C5 --no-cpu --no-e2e --steps 5 > $O/C5_r$m.json 2>&1; done
