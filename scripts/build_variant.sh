#!/bin/bash
# A/B helper: rebuild one unit (SRC=detect by default, e.g. SRC=fullband) with extra nvcc flags and link it with the other
# objects of the normal build into variants/<name>.so (load with HSAD_B200_LIB=...).
#   scripts/build_variant.sh <name> [-DFOO ...]
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
name=$1; shift
mkdir -p "$ROOT/variants/obj_$name"
/usr/local/cuda/bin/nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo \
  -Xcompiler -fPIC -I"$ROOT/include" "$@" -c "$ROOT/paper_1201_2025_b200/csrc/${SRC:-detect}.cu" \
  -o "$ROOT/variants/obj_$name/${SRC:-detect}.o"
SRC=${SRC:-detect}
objs=$(ls "$ROOT"/paper_1201_2025_b200/build/*.o | grep -v "/$SRC.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared \
  -o "$ROOT/variants/$name.so" "$ROOT/variants/obj_$name/${SRC:-detect}.o" $objs -Xcompiler -pthread -ldl
echo "built variants/$name.so"
