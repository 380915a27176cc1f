#!/bin/bash
O=gpurun_out/fs; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_pdl.py tests/test_gpu_parity.py tests/test_gpu_slabs.py -m gpu -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C1 C2 C3; do for f in 1 0; do MG_FUSE_SCALARS=$f timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_f$f.json 2>&1; done; done
