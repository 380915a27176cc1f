#!/bin/bash
# full ncu captures of the top fine kernels (one launch each): C3 march2 CGP/RESTRICT/POST, C4 h8.
O=gpurun_out/$1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
CMD="env MG_HOST_LOOP=1 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu --no-e2e"
CMD4="env MG_HOST_LOOP=1 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > $O/plain3.log 2>&1 && $CMD4 > $O/plain4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"march2_kernel<.int.(3|4|5)," -s 30 -c 3 -o $O/prof_march $CMD > $O/ncu1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"h8_kernel<.int.(1|2|3)," -s 30 -c 3 -o $O/prof_h8 $CMD4 > $O/ncu2.log 2>&1
echo "exit $?" > $O/status.txt
