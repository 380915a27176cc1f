#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
MG_H8_VARIANT=1 timeout 900 python -m pytest tests -m gpu -x -q -k "T3 and (matvec or solve)" > $O/pytest_v1.log 2>&1; echo "exit $?" >> $O/pytest_v1.log
for V in 0 1 2; do for C in C4 C5; do MG_H8_VARIANT=$V timeout 600 python bench.py --config $C --no-cpu --no-e2e --steps 3 > $O/bench_${C}_$V.json 2>&1; done; done
