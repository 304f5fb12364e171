#!/bin/bash
# usage: tools/variants.sh NAME "NVCC DEFINES" ...   -- build libmpg_<NAME>.so variants (here, on CPU)
cd "$(dirname "$0")/.."
B=paper_2311_12818_b200
while [ $# -ge 2 ]; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
    -I include -diag-suppress 177 $2 -o $B/libmpg_$1.so $B/csrc/mpg.cu &
  shift 2
done
wait
ls -la $B/libmpg_*.so
