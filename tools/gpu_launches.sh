#!/bin/bash
# launch lists (host-driven loop so loop kernels are visible) for the given configs
O=gpurun_out/launch4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
for C in "$@"; do
CMD="python bench.py --config $C --steps 1 --warmup 3 --no-cpu --no-e2e"
MG_HOST_LOOP=1 $CMD > $O/plain_$C.log 2>&1 && \
MG_HOST_LOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 6000 --csv --log-file $O/launches_$C.csv $CMD > $O/ncu_$C.log 2>&1
done
