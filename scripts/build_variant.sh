#!/bin/bash
# Build a timing-experiment variant of the library: kernels.cu compiled with
# extra -D flags, linked with the normal objects into libigm_<name>.so
# (used with LIBNAME=libigm_<name>.so by scripts/tile_bench.py).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -fmad=false -Iinclude "$@" \
  -c paper_2009_07495_b200/csrc/kernels.cu -o build/kernels_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2009_07495_b200/libigm_$name.so build/kernels_$name.o \
  build/setup.o build/capi.o build/shim.o build/schedule.o build/mm_io.o build/experiment.o
