#!/bin/bash
# bench lines only: default (C3 + cpu_baseline + e2e), reference arm, C1, C2, C4, C5 (with e2e)
O=gpurun_out/$1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/status.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench exit $?" >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref exit $?" >> $O/status.txt
for C in C1 C2 C4 C5; do timeout 600 python bench.py --config $C --no-cpu --steps 5 > $O/bench_$C.json 2>&1; done
