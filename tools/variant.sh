#!/bin/bash
# Kernel-variant build for A/B runs: recompile one source with extra -D flags
# and link it with the other objects into build/var/<name>/libfvlog.so, to be
# loaded with FVLOG_LIB=build/var/<name>/libfvlog.so.
#   bash tools/variant.sh <name> <source.cu> "<flags>"
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; flags=$3
make -s all
d=build/var/$name; mkdir -p $d
base=$(basename $src .cu)
NV="/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -ccbin /usr/bin/g++ -Xcompiler -fPIC -Iinclude -Ipaper_2501_13051_b200/csrc --expt-relaxed-constexpr"
$NV $flags -c paper_2501_13051_b200/csrc/$base.cu -o $d/$base.o
objs=$(ls build/obj/*.o | grep -v "/$base.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -ccbin /usr/bin/g++ -shared -o $d/libfvlog.so $objs $d/$base.o -cudart static -lpthread
echo "$d/libfvlog.so"
