#!/bin/bash
# launch list + full ncu capture for one config. usage: bash tools/gpu_prof.sh <tag> <config> <kernel regex> [skip]
TAG=$1; C=$2; K=$3; S=${4:-20}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
CMD="python bench.py --config $C --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 4 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "exit $?" > $O/status.txt
