#!/bin/bash
O=gpurun_out/ns5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
for i in 1 2 3; do
timeout 300 python bench.py --config C3 --no-cpu --no-e2e --steps 8 >> $O/C3_default.json 2>&1
MG_LIB=$PWD/paper_1909_13585_b200/_libvar/ns5.so timeout 300 python bench.py --config C3 --no-cpu --no-e2e --steps 8 >> $O/C3_ns5.json 2>&1
done
for i in 1 2; do
timeout 300 python bench.py --config C2 --no-cpu --no-e2e --steps 8 >> $O/C2_default.json 2>&1
MG_LIB=$PWD/paper_1909_13585_b200/_libvar/ns5.so timeout 300 python bench.py --config C2 --no-cpu --no-e2e --steps 8 >> $O/C2_ns5.json 2>&1
done
