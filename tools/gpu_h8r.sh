#!/bin/bash
# plane-ring H8 kernel incl. fused RESTR3: 3D parity tests + A/B
O=gpurun_out/h8r3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_wilson.py -m gpu -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for C in C5 C4; do for f in 0 1 3; do
MG_FUSED3D=$f timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_f$f.json 2>&1
done
MG_FUSED3D=1 MG_H8_VARIANTS=-1,-1,-1,-1,0 timeout 300 python bench.py --config $C --no-cpu --no-e2e --steps 5 > $O/${C}_f1_old.json 2>&1
done
