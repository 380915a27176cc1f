#!/bin/bash
O=gpurun_out/gjp7; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modes.py -m gpu -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C5 C4 C3; do timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}.json 2>&1; done
CMD="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gj_" -c 400 --csv --log-file $O/gj.csv $CMD > $O/ncu.log 2>&1
