#!/bin/bash
# Build a variant library from the current csrc with some files taken from a
# git revision:  tools/build_rev_variant.sh NAME REV file1[@rev1] [file2 ...]
# (paths relative to paper_2506_15704_b200/csrc; file@rev overrides REV)
# -> lib/variants/NAME.so
set -e
name=$1; rev=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=/tmp/lfps_rev_$name
rm -rf "$tmp"; mkdir -p "$tmp/csrc" "$tmp/include"
cp "$root"/paper_2506_15704_b200/csrc/*.cu "$root"/paper_2506_15704_b200/csrc/*.cuh "$tmp/csrc/"
cp "$root"/include/*.h "$tmp/include/"
# common.cuh includes ../../include/lfps_b200.h
mkdir -p "$tmp/a/b"; mv "$tmp/csrc" "$tmp/a/b/csrc"; mv "$tmp/include" "$tmp/a/include"
for spec in "$@"; do
  f=${spec%@*}; r=$rev
  [ "$spec" != "$f" ] && r=${spec#*@}
  git -C "$root" show "$r:paper_2506_15704_b200/csrc/$f" > "$tmp/a/b/csrc/$f"
done
mkdir -p "$root/paper_2506_15704_b200/lib/variants"
objs=()
for f in "$tmp"/a/b/csrc/*.cu; do
  o=${f%.cu}.o
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
       -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -c "$f" -o "$o" &
  objs+=("$o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/paper_2506_15704_b200/lib/variants/$name.so" "${objs[@]}" -lcudart
echo "$root/paper_2506_15704_b200/lib/variants/$name.so"
