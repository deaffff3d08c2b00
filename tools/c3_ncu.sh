#!/usr/bin/env bash
# ncu capture of the C3 wide step kernel (one launch), exported on the box as
# raw + SASS-source CSV (tools/sass_lines.py joins them with nvdisasm line info).
# usage: tools/c3_ncu.sh TAG
set -u
TAG=${1:-r02x}
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:step_kernel \
  --launch-skip 2 --launch-count 1 -o /tmp/c3step -f python tools/c3_run.py --iters 4 > $O/${TAG}_c3ncu.log 2>&1
ncu -i /tmp/c3step.ncu-rep --page raw --csv > $O/${TAG}_c3step_raw.csv 2>&1
ncu -i /tmp/c3step.ncu-rep --page source --csv --print-source sass > $O/${TAG}_c3step_sass.csv 2>&1
