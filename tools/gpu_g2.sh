#!/bin/bash
O=gpurun_out/g3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "stress" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for i in 1 2; do timeout 600 python bench.py --config C3 --no-cpu --steps 5 >> $O/C3.json 2>&1; done
