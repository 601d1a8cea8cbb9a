#!/bin/bash
# Build paper_2601_15013_b200/_rdx_<tag>.so with csrc/<file> taken from git revision <rev>
# (everything else from the working tree): A/B of one kernel in one process.
#   scripts/build_variant.sh <tag> <rev> <file>      e.g. base HEAD~1 attention.cu
set -e
tag=$1; rev=$2; file=$3
root=$(cd "$(dirname "$0")/.." && pwd)
base=$(mktemp -d)
tmp=$base/pkg/csrc   # common.cuh includes ../../include/radix_b200.h
mkdir -p "$tmp"
ln -s "$root/include" "$base/include"
cp "$root"/paper_2601_15013_b200/csrc/* "$tmp"/
git -C "$root" show "$rev:paper_2601_15013_b200/csrc/$file" > "$tmp/$file"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -diag-suppress 177 -I "$root/include" -o "$root/paper_2601_15013_b200/_rdx_$tag.so" "$tmp"/*.cu
rm -rf "$base"
echo "built _rdx_$tag.so ($file from $rev)"
