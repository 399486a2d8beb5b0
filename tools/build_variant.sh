#!/bin/bash
# Build a design/debug variant of the library: tools/build_variant.sh <name> [-D...]
#   phase: -DDIALSORT_PHASE_MARKS=1 (per-phase %globaltimer stamps, tools/phase_times.py)
# Loaded with DIALSORT_LIB_VARIANT=<name> (development only; the product is libdialsort.so).
set -e
name=$1; shift
[ "$name" = phase ] && [ $# -eq 0 ] && set -- -DDIALSORT_PHASE_MARKS=1
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -shared -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 \
  "$@" -o paper_2605_16667_b200/libdialsort_$name.so paper_2605_16667_b200/csrc/dialsort.cu
