#!/bin/bash
# Sort-kernel variant build for A/B runs of tools/sortbench.cu: radix_sort.cu
# recompiled with extra -D flags into build/var/sort_<name>/sortbench.
#   bash tools/sortvar.sh <name> "<flags>"
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2
make -s all
d=build/var/sort_$name; mkdir -p $d
NV="/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -ccbin /usr/bin/g++ -Xcompiler -fPIC -Iinclude -Ipaper_2501_13051_b200/csrc --expt-relaxed-constexpr"
$NV $flags -Xptxas -v -c paper_2501_13051_b200/csrc/radix_sort.cu -o $d/radix_sort.o 2> $d/ptxas.txt
$NV -o $d/sortbench tools/sortbench.cu build/obj/fv_ctx.o build/obj/prim.o $d/radix_sort.o -cudart static -lpthread
echo "$d/sortbench"
