#!/usr/bin/env bash
# Build the whole product library of another git revision into
# build/var_<name>.so (A/B against the working tree with tools/ab.sh):
#   bash tools/build_revision.sh HEAD~1 prev
set -eu
cd "$(dirname "$0")/.."
rev=$1; name=$2
src=$(mktemp -d)
git archive "$rev" paper_1403_1706_b200/csrc include | tar -x -C "$src"
mkdir -p "$src/obj" build
for f in "$src"/paper_1403_1706_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I"$src/include" -c -o "$src/obj/$(basename "$f" .cu).o" "$f" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "build/var_$name.so" "$src"/obj/*.o
rm -rf "$src"
echo "build/var_$name.so"
