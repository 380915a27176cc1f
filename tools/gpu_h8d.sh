#!/bin/bash
O=gpurun_out/h8d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q -k "T3 or C4 or C5" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
bash tools/gpu_ab.sh h8d_ab4 C4
bash tools/gpu_ab.sh h8d_ab5 C5
