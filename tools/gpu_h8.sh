#!/bin/bash
O=gpurun_out/h8a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "T3 or C4 or slab" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for C in C4 C5; do timeout 600 python bench.py --config $C --no-cpu --no-e2e --steps 3 > $O/bench_$C.json 2>&1; done
CMD="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > $O/ncu_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:h8_kernel -s 20 -c 2 -o $O/prof $CMD > $O/ncu.log 2>&1
echo "ncu exit $?" >> $O/pytest.log
