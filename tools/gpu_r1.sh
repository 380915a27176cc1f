#!/bin/bash
# One gpurun session: GPU parity tests, bench lines, ncu launch list + full capture.
# usage (under gpurun): bash tools/gpu_r1.sh <tag> [ncu_kernel_regex] [ncu_config]
set -u
TAG=${1:-r1}
KREG=${2:-march2}
NCFG=${3:-C3}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
for C in C3 C5 C4 C2 C1; do
  X=""; [ $C != C3 ] && X="--no-cpu"
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 $X > $O/bench_$C.json 2> $O/bench_$C.err
  echo "$C exit $?" >> $O/bench_status.txt
done
CMD="python bench.py --config $NCFG --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > $O/ncu_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KREG -s 30 -c 3 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "ncu exit $?" >> $O/bench_status.txt
