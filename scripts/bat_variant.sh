#!/bin/bash
# build a standalone profiling variant of binattn_tc.cu with extra -D flags: bat_variant.sh OUT.so FLAGS...
out=$1; shift
cd "$(dirname "$0")/../paper_2306_06446_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DBAT_PROF "$@" -shared -I../../include -I. binattn_tc.cu lib.cu -o "$out"
