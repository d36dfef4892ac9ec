#!/bin/bash
# Build a variant of liblfps_b200.so with extra nvcc defines into
# paper_2506_15704_b200/lib/variants/<name>.so (select it with LFPS_LIB=...).
#   tools/build_variant.sh s2 -DLFPS_ROW_STAGES=2
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_2506_15704_b200/csrc
out=$root/paper_2506_15704_b200/lib/variants
mkdir -p "$out" "/tmp/lfps_variant_$name"
objs=()
for f in "$src"/*.cu; do
  o=/tmp/lfps_variant_$name/$(basename "$f" .cu).o
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
       -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr "$@" -c "$f" -o "$o" &
  objs+=("$o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/$name.so" "${objs[@]}" -lcudart
echo "$out/$name.so"
