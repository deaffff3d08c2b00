#!/usr/bin/env bash
# One ncu --set full capture of a kernel of the C5 bench, exported on the box
# as raw + SASS-source CSV (the report itself can exceed gpurun's copy-back).
# usage: tools/ncu_kernel_csv.sh TAG KERNEL_REGEX LAUNCH_SKIP
set -u
TAG=$1; RX=$2; SKIP=${3:-5}
O=gpurun_out; mkdir -p $O
SHORT="--steps 2 --warmup 3 --no-c1 --no-c3 --no-cpu-baseline --no-converge"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:$RX \
  --launch-skip $SKIP --launch-count 1 -o /tmp/${TAG}_k -f python bench.py $SHORT > $O/${TAG}_ncu.log 2>&1
ncu -i /tmp/${TAG}_k.ncu-rep --page raw --csv > $O/${TAG}_raw.csv 2>&1
ncu -i /tmp/${TAG}_k.ncu-rep --page source --csv --print-source sass > $O/${TAG}_sass.csv 2>&1
