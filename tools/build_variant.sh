#!/bin/bash
# Build a variant of the library into altlib/NAME/ (development A/B):
#   tools/build_variant.sh NAME [-DFLAG=...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p altlib/$name
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off -shared -diag-suppress 550 "$@" \
  -o altlib/$name/libpch_b200.so paper_1305_1293_b200/csrc/pch_engine.cu paper_1305_1293_b200/csrc/pch_mesh.cpp
echo altlib/$name/libpch_b200.so
