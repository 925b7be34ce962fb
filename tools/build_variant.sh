#!/bin/bash
# Build libdeltanet from a source tree (default: the working tree) into OUT,
# with extra nvcc flags (profiling aid for tools/ab_time.py).
#   tools/build_variant.sh OUT.so [SRC_DIR] [extra nvcc flags...]
set -e
OUT=$1; SRC=${2:-paper_2406_06484_b200/csrc}; shift; shift || true
ROOT=$(cd "$(dirname "$0")/.." && pwd)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -shared -I "$ROOT/include" "$@" -o "$OUT" "$SRC"/*.cu
