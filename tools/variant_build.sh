#!/bin/bash
# Build a tuning variant of the library: one CUDA source recompiled with extra -D flags, linked
# with the regular objects into variants/<name>/libpencil_b200.so (select it at run time with
# PENCIL_B200_LIB=...).  Usage: tools/variant_build.sh <name> <k_source.cu> -DMACRO=V ...
set -e
name=$1; src=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
pkg=$root/paper_1302_5586_b200
out=$root/variants/$name
mkdir -p "$out"
ARCH="-gencode arch=compute_100a,code=sm_100a"
base=$(basename "$src" .cu)
/usr/local/cuda/bin/nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr \
    "$@" -c "$pkg/csrc/$base.cu" -o "$out/$base.o" 2> "$out/$base.ptxas.log"
objs=$(ls $pkg/build/*.o | grep -v "/$base.o$")
/usr/local/cuda/bin/nvcc $ARCH -shared -o "$out/libpencil_b200.so" $objs "$out/$base.o" -cudart static \
    -Xlinker --no-undefined -lpthread -ldl -lrt
echo "$out/libpencil_b200.so"
