#!/bin/bash
O=gpurun_out/dam; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py tests/test_gpu_block.py tests/test_gpu_slabs.py tests/test_gpu_sens.py -m gpu -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C2 C3 C4 C1; do for m in 1 0; do
MG_DENSE_MMA=$m timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_m$m.json 2>&1
done; done
