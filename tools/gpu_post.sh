#!/bin/bash
O=gpurun_out/post; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_fullsize.py -m gpu -x -q -k "T2 or C1 or C2 or C3" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C3 C2; do timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_default.json 2>&1
for f in paper_1909_13585_b200/_libvar/*.so; do n=$(basename $f .so); MG_LIB=$PWD/$f timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_$n.json 2>&1; done; done
