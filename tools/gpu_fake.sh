#!/bin/bash
O=gpurun_out/fake2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
CMD="python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e"
MG_HOST_LOOP=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none -k regex:"coarse_kernel" -c 40 --csv --log-file $O/default.csv $CMD > $O/ncu_default.log 2>&1
MG_LIB=$PWD/paper_1909_13585_b200/_libvar/fakehalf.so MG_HOST_LOOP=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none -k regex:"coarse_kernel" -c 40 --csv --log-file $O/fakehalf.csv $CMD > $O/ncu_fakehalf.log 2>&1
