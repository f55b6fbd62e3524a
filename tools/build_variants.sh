#!/bin/bash
# Build experimental variants of the kernel library into tools/variants/ (dev only):
# every CUDA source compiled with the extra flags, the C++ sources as usual.
set -e
cd "$(dirname "$0")/../paper_1903_07189_b200/csrc"
mkdir -p ../../tools/variants
CXXF="-O2 -fPIC -std=c++17 -ffp-contract=off -fno-fast-math -fvisibility=hidden -I/usr/local/cuda/include"
g++ $CXXF -c -o /tmp/v_synth.o synth.cpp
g++ $CXXF -c -o /tmp/v_shard.o wmc_shard.cpp
g++ $CXXF -c -o /tmp/v_ipc.o wmc_ipc.cpp
for v in "$@"; do
  name=$(echo "$v" | tr ' =' '_-')
  objs=""
  for src in wmc_capi wmc_io wmc_reduce wmc_f64; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
         -Xcompiler -fPIC,-fvisibility=hidden $v -c -o /tmp/v_${name}_$src.o $src.cu 2>/dev/null
    objs="$objs /tmp/v_${name}_$src.o"
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/variants/lib_$name.so $objs \
       /tmp/v_synth.o /tmp/v_shard.o /tmp/v_ipc.o -lpthread
  echo built $name
done
