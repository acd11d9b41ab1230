#!/bin/bash
# Debug build with per-phase clock64 timers (-DHSAD_PHASE_TIMERS) -> libhsad_b200_pt.so
set -e
cd "$(dirname "$0")/../paper_1201_2025_b200"
mkdir -p build_pt
for f in csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -Xcompiler -fPIC -I../include -DHSAD_PHASE_TIMERS -c "$f" -o "build_pt/$(basename "$f" .cu).o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libhsad_b200_pt.so build_pt/*.o
