#!/bin/bash
# Dev: build an A/B variant of libsshgpu.so from csrc with sed edits applied.
# usage: scripts/build_variant.sh OUT.so 'sed-expr-for-FILE' FILE [...]
set -e
out=$1; shift
tmp=$(mktemp -d)
root=$(cd "$(dirname "$0")/.." && pwd)
cp -r "$root/paper_1610_07328_b200/csrc/." "$tmp/"
sed -i "s#../../include/sshgpu.h#$root/include/sshgpu.h#" "$tmp/common.cuh"
while [ $# -ge 2 ]; do sed -i "$1" "$tmp/$2"; shift 2; done
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared --cudart static \
  -I "$(dirname "$0")/../include" -o "$out" "$tmp"/*.cu
rm -rf "$tmp"
