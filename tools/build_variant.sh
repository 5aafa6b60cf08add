#!/bin/bash
# Build an A/B variant of libmlb with extra -D flags on ONE source file, linked
# with the other objects of the last in-tree build:
#   tools/build_variant.sh <name> <source.cu> -DFOO=1 ...  ->  paper_2007_05239_b200/libmlb_<name>.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; src=$2; shift 2
B=$ROOT/build/mlb; V=$ROOT/build/var_$name; mkdir -p $V
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O2 \
  --expt-relaxed-constexpr -I $ROOT/include "$@" -c $ROOT/paper_2007_05239_b200/csrc/$src -o $V/$src.o
objs=$(ls $B/*.o | grep -v "/$src.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/paper_2007_05239_b200/libmlb_$name.so $objs $V/$src.o -lcudart
echo built libmlb_$name.so
