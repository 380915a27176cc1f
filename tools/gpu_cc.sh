#!/bin/bash
O=gpurun_out/cc; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_modes.py -m gpu -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
MG_UNFUSED_COARSE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "vcycle or solve_parity" > $O/tests_unfused.log 2>&1; echo "rc=$?" >> $O/tests_unfused.log
for C in C4 C5; do for m in 1 0; do
MG_COARSE_COMP=$m timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_m$m.json 2>&1
done; done
