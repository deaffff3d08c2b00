#!/usr/bin/env bash
# Round-end GPU pass: tests, reference suite, bench, the ncu launch list and one
# --set full capture of each of the three hot kernels exported as CSV.
# usage: tools/final_round.sh TAG
set -u
TAG=${1:-r02z}
O=gpurun_out
bash tools/gpu_round.sh $TAG tests refsuite bench launches
bash tools/ncu_kernel_csv.sh ${TAG}_probe probe_split 3
bash tools/ncu_kernel_csv.sh ${TAG}_commit commit_kernel 3
bash tools/ncu_kernel_csv.sh ${TAG}_factor factor_grads 5
rm -f $O/*_sass.csv.tmp
