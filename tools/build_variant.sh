#!/bin/bash
# Build libhx with extra nvcc defines into build/variants/<name>/libhx.so (A/B runs:
# HX_LIB=build/variants/<name>/libhx.so python tools/kernel_bench.py ...).
#   tools/build_variant.sh poly4 -DHX_POLY_EVERY=4
set -e
name=$1; shift
out=build/variants/$name
mkdir -p $out
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
     --expt-relaxed-constexpr -Iinclude "$@" -shared -o $out/libhx.so paper_2507_00394_b200/csrc/*.cu
echo $out/libhx.so
