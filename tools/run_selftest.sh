#!/bin/bash
# Build and run the kernel self-test (on the GPU box).
set -e
cd "$(dirname "$0")/.."
B=paper_2206_12409_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -Iinclude -o $B/kernel_selftest tools/kernel_selftest.cu \
  $B/ttapply.cu.o $B/linalg.cu.o $B/entries.cu.o $(ls $B/crosskern.cu.o 2>/dev/null) -cudart static
./$B/kernel_selftest
