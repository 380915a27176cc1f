#!/bin/bash
O=gpurun_out/pdlsafe; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
for i in 1 2; do timeout 1200 python -m pytest tests -m gpu -q > $O/tests_$i.log 2>&1; echo "rc=$?" >> $O/tests_$i.log; done
