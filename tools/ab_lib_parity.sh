#!/usr/bin/env bash
# tools/ab_lib.sh plus the C5/C2/C1 parity tests under each variant library.
# Usage: tools/ab_lib_parity.sh TAG var_a var_b ...
O=gpurun_out
TAG=$1
bash tools/ab_lib.sh "$@"
shift
for V in "$@"; do
  mkdir -p $O/${TAG}_$V.dump
  GVP_B200_LIB=paper_2411_03416_b200/$V/libgvp_b200.so GVP_PARITY_DUMP=$O/${TAG}_$V.dump timeout 900 \
    python -m pytest tests/test_gpu_trace_parity.py tests/test_gpu_engine.py tests/test_gpu_c4.py -q -s \
    -p no:cacheprovider > $O/${TAG}_${V}_tests.log 2>&1
  echo "rc=$?" >> $O/${TAG}_${V}_tests.log
done
