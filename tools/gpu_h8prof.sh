#!/bin/bash
O=gpurun_out/h8p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
CMD="python bench.py --config C4 --steps 1 --warmup 3 --no-cpu --no-e2e"
MG_HOST_LOOP=1 $CMD > $O/plain.log 2>&1 && \
MG_HOST_LOOP=1 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"h8r_kernel|h8_kernel" -s 40 -c 3 -o $O/prof $CMD > $O/ncu.log 2>&1
echo "exit $?" >> $O/ncu.log
