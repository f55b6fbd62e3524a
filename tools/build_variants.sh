#!/bin/bash
# Build experimental variants of the kernel library into tools/variants/ (dev only).
set -e
cd "$(dirname "$0")/../paper_1903_07189_b200/csrc"
mkdir -p ../../tools/variants
for v in "$@"; do
  name=$(echo "$v" | tr ' =' '_-')
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
       -Xcompiler -fPIC,-fvisibility=hidden $v -c -o /tmp/v_$name.o wmc_capi.cu 2>/dev/null
  g++ -O2 -fPIC -std=c++17 -ffp-contract=off -fvisibility=hidden -c -o /tmp/v_synth.o synth.cpp
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/variants/lib_$name.so /tmp/v_$name.o /tmp/v_synth.o
  echo built $name
done
