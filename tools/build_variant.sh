#!/bin/bash
# Builds an experimental variant of libqgpu.so with extra -D flags:
#   tools/build_variant.sh <name> -DQGPU_PHASE_REG_BITS=3
# -> paper_1802_08032_b200/_lib/libqgpu_<name>.so (select with QGPU_LIB=...)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=paper_1802_08032_b200/_lib/var_$name; mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="-O3 -std=c++20 -lineinfo --fmad=false -Xcompiler -fPIC,-O3,-ffp-contract=off -Xcicc -jump-table-density=1 -Iinclude -Ipaper_1802_08032_b200/csrc $@"
for s in kernels.cu tile_pass.cu runtime.cpp api.cpp transport.cpp memory_plan.cpp swap_plan.cpp tile_jit.cpp; do
  lang=c++; [[ $s == *.cu ]] && lang=cu
  /usr/local/cuda/bin/nvcc $ARCH $FLAGS -x $lang -c paper_1802_08032_b200/csrc/$s -o $out/${s%.*}.o &
done
wait
/usr/local/cuda/bin/nvcc $ARCH -shared -o paper_1802_08032_b200/_lib/libqgpu_$name.so $out/*.o -ldl -lpthread
echo paper_1802_08032_b200/_lib/libqgpu_$name.so
