#!/bin/bash
O=gpurun_out/2dt; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "T2 or C1 or C2 or slab or wilson" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
bash tools/gpu_ab.sh 2dt_ab C3
