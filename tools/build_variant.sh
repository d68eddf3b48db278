#!/bin/bash
# build an experiment variant of libhegrid.so: tools/build_variant.sh NAME -DFOO=1 ...
name=$1; shift
mkdir -p tmp_libs
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O2 -shared --expt-relaxed-constexpr -cudart static "$@" -o tmp_libs/lib_$name.so paper_2207_04584_b200/csrc/*.cu -lpthread && echo built tmp_libs/lib_$name.so
