#!/bin/bash
O=gpurun_out/j6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
MG_H8_VARIANTS=-1,-1,6,-1,-1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "T3" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C5 C4; do for v in "-1,-1,-1,-1,-1" "-1,-1,6,-1,-1" "-1,-1,4,-1,-1"; do
MG_H8_VARIANTS=$v timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_${v//,/_}.json 2>&1
done; done
