#!/usr/bin/env bash
# Build a variant of the product library with extra -D flags on one source
# (A/B experiments on the GPU box via QGM_LIB=build/var_<name>.so):
#   bash tools/build_variant.sh <name> <source.cu> -DQGM_JOIN_DRAIN=32 ...
# <source.cu> is a file of paper_1403_1706_b200/csrc, or a path to another
# copy of one (e.g. an older revision: git show REV:path > build/src/x.cu)
set -eu
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
make -s lib >/dev/null
mkdir -p build/var
objs=$(ls build/obj/*.o | grep -v "/$(basename $src .cu).o")
[ -f "$src" ] || src=paper_1403_1706_b200/csrc/$src
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Iinclude -Ipaper_1403_1706_b200/csrc "$@" -c -o build/var/$name.o $src
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$name.so $objs build/var/$name.o
echo build/var_$name.so
