#!/usr/bin/env bash
# Build a variant of libgvp_b200.so with one source file recompiled under extra
# defines, for A/B runs on the GPU box (GVP_B200_LIB=<out>/libgvp_b200.so).
# Usage: tools/variant_build.sh <csrc file stem> <outdir under paper_2411_03416_b200/> <-Dflags...>
set -e
cd "$(dirname "$0")/.."
stem=$1; tag=$2; out=paper_2411_03416_b200/$2; shift 2
mkdir -p build_var/$tag "$out"
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3 \
  --expt-relaxed-constexpr "$@" -c paper_2411_03416_b200/csrc/$stem.cu -o build_var/$tag/$stem.o
objs=$(ls build/*.o | grep -v "/$stem.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libgvp_b200.so" \
  $objs build_var/$tag/$stem.o -Xcompiler -fPIC
echo "built $out/libgvp_b200.so"
