#!/bin/bash
# Development tool: build libvolkrig_b200.so with extra nvcc flags for one
# translation unit into variants/<name>/ (the in-tree library is untouched).
#   tools/build_variant.sh <name> <unit.cu> [nvcc flags...]
set -e
cd "$(dirname "$0")/.."
name=$1; unit=$2; shift 2
N=paper_2303_09523_b200/_native; C=paper_2303_09523_b200/csrc
mkdir -p variants/$name
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I include -I $C "$@" -c $C/$unit -o variants/$name/$unit.o
objs=""
for o in $N/*.o; do b=$(basename $o); if [ "$b" = "$unit.o" ]; then objs="$objs variants/$name/$unit.o"; else objs="$objs $o"; fi; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name/libvolkrig_b200.so $objs -cudart static -ldl
echo variants/$name/libvolkrig_b200.so
