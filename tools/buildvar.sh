#!/bin/bash
# Build a variant of libmgcg.so with extra nvcc flags for one source file (A/B on the GPU box:
# MG_LIB=paper_1909_13585_b200/_libvar/<name>.so python bench.py ...).
#   tools/buildvar.sh <name> <file.cu> "<nvcc flags>" [replaced object: default <file>.o]
set -e
cd "$(dirname "$0")/../paper_1909_13585_b200/csrc"
make -s -j16 >/dev/null
name=$1; src=$2; flags=$3; base=${4:-${src%.cu}}
mkdir -p build/var ../_libvar
obj=build/var/${name}_${src%.cu}.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -I$(python3 -c 'import nvidia.nccl, os; print(os.path.join(list(nvidia.nccl.__path__)[0], "include"))') \
  -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Xptxas -v $flags -c $src -o $obj 2> build/var/${name}.ptxas.log
objs=$(ls build/*.o | grep -v "build/${base}.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../_libvar/${name}.so $objs $obj -cudart static -ldl
echo built ../_libvar/${name}.so
