#!/usr/bin/env bash
# A/B of library variants (tools/variant_build.sh) on C5: short bench runs, the
# default library first. Usage: tools/ab_lib.sh TAG var_a var_b ...
O=gpurun_out
TAG=$1; shift
SHORT="--steps 10 --warmup 3 --no-c1 --no-c3 --no-cpu-baseline --no-converge"
timeout 300 python bench.py $SHORT > $O/${TAG}_default.json 2>&1
for V in "$@"; do
  GVP_B200_LIB=paper_2411_03416_b200/$V/libgvp_b200.so timeout 300 python bench.py $SHORT > $O/${TAG}_$V.json 2>&1
done
