#!/bin/bash
# final evidence: smoke, full GPU suite, bench lines (default + reference + C1/C2/C4/C5), launch lists C3/C5,
# ncu --set full of the C3 march2 kernels
O=gpurun_out/$1; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/status.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/tests_gpu.log 2>&1; echo "tests exit $?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench exit $?" >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref exit $?" >> $O/status.txt
for C in C1 C2 C4 C5; do timeout 600 python bench.py --config $C --no-cpu --steps 5 > $O/bench_$C.json 2>&1; done
CMD="env MG_HOST_LOOP=1 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu --no-e2e"
CMD5="env MG_HOST_LOOP=1 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > $O/plain3.log 2>&1 && $CMD5 > $O/plain5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 6000 --csv --log-file $O/launches_C3.csv $CMD > $O/ncu1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 6000 --csv --log-file $O/launches_C5.csv $CMD5 > $O/ncu2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"march2_kernel<.int.(3|4|5)," -s 30 -c 3 -o $O/prof_march $CMD > $O/ncu3.log 2>&1
echo "ncu exit $?" >> $O/status.txt
