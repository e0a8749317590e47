#!/bin/bash
# usage: tools/sass_stats.sh <src.cu> <kernel-substring>  -> ptxas -v summary + SASS of the kernel in /tmp/k.sass
set -e
cd "$(dirname "$0")/.."
src=$1; pat=$2
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xptxas -v -std=c++17 -diag-suppress 177 \
  -Iinclude -c "$src" -o /tmp/k.o 2>&1 | grep -E 'error|registers|spill' || true
cuobjdump -sass /tmp/k.o | awk -v p="$pat" '/Function :/{f=index($0,p)>0} f' > /tmp/k.sass
wc -l < /tmp/k.sass
