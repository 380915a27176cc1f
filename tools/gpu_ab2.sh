#!/bin/bash
O=gpurun_out/$1; mkdir -p $O; C=${2:-C3}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_default.json 2>&1
for f in paper_1909_13585_b200/_libvar/*.so; do n=$(basename $f .so); MG_LIB=$PWD/$f timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_$n.json 2>&1; done
