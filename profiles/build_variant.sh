#!/bin/bash
# Build libmhg.so with extra nvcc defines into variants/libmhg_<name>.so (A/B only).
# usage: profiles/build_variant.sh name -DFOO=1 ...
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_1705_04807_b200/csrc
mkdir -p $R/variants /tmp/mhg_variant_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$R/include -I$C "$@" \
     -Xptxas -v -c $C/mhg_kernels.cu -o /tmp/mhg_variant_$name/k.o 2> /tmp/mhg_variant_$name/ptxas.log
grep -A2 "k_gemmILi2" /tmp/mhg_variant_$name/ptxas.log | grep -E "spill|registers" | sed "s/^/[$name] /"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/variants/libmhg_$name.so /tmp/mhg_variant_$name/k.o \
     $C/build/mhg_host.o $C/build/mhg_planner.o $C/build/mhg_wire.o $C/build/mhg_options.o -lcudart_static -lrt -lpthread -ldl
