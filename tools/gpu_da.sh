#!/bin/bash
O=gpurun_out/da2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "vcycle or coarse_inverse or solve_parity" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C5 C4 C3 C2; do timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_default.json 2>&1
MG_LIB=$PWD/paper_1909_13585_b200/_libvar/da_old.so timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_old.json 2>&1; done
CMD="python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"dense_apply" -c 20 --csv --log-file $O/da.csv $CMD > $O/ncu.log 2>&1
