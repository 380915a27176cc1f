#!/bin/bash
O=gpurun_out/gjd2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "coarse_inverse or galerkin or solve_parity" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C2 C3 C4; do timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_default.json 2>&1
MG_LIB=$PWD/paper_1909_13585_b200/_libvar/gjhead.so timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_head.json 2>&1; done
CMD="python bench.py --config C2 --steps 1 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"gj_" -c 200 --csv --log-file $O/gj.csv $CMD > $O/ncu.log 2>&1
