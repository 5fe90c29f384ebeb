#!/bin/bash
# Build an experiment variant of the engine: engine.cu recompiled with extra -D
# flags, linked with the default build's other objects, into lib/libtreeserve_b200_<name>.so.
#   tools/build_variant.sh <name> -DTS_HEAVY_WARPS=6 -DTS_HEAVY_MINB=3
# Load it with TS_LIB_PATH=paper_2604_00510_b200/lib/libtreeserve_b200_<name>.so.
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
L=$R/paper_2604_00510_b200/lib
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC \
  -I "$R/include" "$@" -c -o "$L/engine_$name.o" "$R/paper_2604_00510_b200/csrc/engine.cu"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$L/libtreeserve_b200_$name.so" \
  "$L/engine_$name.o" "$L/policy.o" "$L/beam.o" "$L/steps.o"
