#!/usr/bin/env bash
# Diagnostic build of the probe kernel with per-role work/wait cycle counters
# (-DGVP_PROBE_PROFILE) linked with the regular objects into
# paper_2411_03416_b200/prof/libgvp_b200.so (GVP_B200_LIB selects it).
set -e
cd "$(dirname "$0")/.."
mkdir -p build_prof paper_2411_03416_b200/prof
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3 \
  --expt-relaxed-constexpr -DGVP_PROBE_PROFILE -c paper_2411_03416_b200/csrc/step_probe.cu -o build_prof/step_probe.o
objs=$(ls build/*.o | grep -v step_probe.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2411_03416_b200/prof/libgvp_b200.so \
  $objs build_prof/step_probe.o -Xcompiler -fPIC
