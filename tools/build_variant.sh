#!/usr/bin/env bash
# Build a variant of the product library with extra -D flags on one source
# (A/B experiments on the GPU box via QGM_LIB=build/var_<name>.so):
#   bash tools/build_variant.sh <name> <source.cu> -DQGM_JOIN_DRAIN=32 ...
set -eu
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
make -s lib >/dev/null
mkdir -p build/var
objs=$(ls build/obj/*.o | grep -v "/$(basename $src .cu).o")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Iinclude "$@" -c -o build/var/$name.o paper_1403_1706_b200/csrc/$src
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$name.so $objs build/var/$name.o
echo build/var_$name.so
