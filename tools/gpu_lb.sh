#!/bin/bash
O=gpurun_out/lb; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_modes.py -m gpu -x -q -k "T3 or 3d or modes or C4" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
MG_UNFUSED_COARSE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "vcycle or solve_parity" > $O/tests_unf.log 2>&1; echo "rc=$?" >> $O/tests_unf.log
for C in C5 C4; do timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}.json 2>&1; done
