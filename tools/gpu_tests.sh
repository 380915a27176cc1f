#!/bin/bash
# GPU test session: build, gpu tests (optionally a -k filter), smoke. usage: bash tools/gpu_tests.sh <tag> [pytest -k expr]
TAG=${1:-t}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; tail -20 $O/build.log; exit 1; }
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 1500 python -m pytest tests -m gpu -x -q $K > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -30 $O/pytest_gpu.log
