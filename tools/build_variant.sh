#!/usr/bin/env bash
# Tuning builds of the library with extra defines, only the C4 / shard / C2 shapes:
#   bash tools/build_variant.sh OUT.so -DVPM_PHASE_TIMING ...
set -euo pipefail
OUT=$1; shift
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -fmad=false -shared -Xcompiler -fPIC \
  -DVPM_TUNING_SUBSET "$@" paper_2509_16079_b200/csrc/vpm_capi.cu -o "$OUT"
