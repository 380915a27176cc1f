#!/bin/bash
O=gpurun_out/pdl3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/build.log 2>&1 || { echo "build/smoke failed" >> $O/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "T3 or h8 or T2 or C1" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C4 C5 C2 C1; do for p in 1 0; do
MG_PDL=$p timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_p$p.json 2>&1
done; done
