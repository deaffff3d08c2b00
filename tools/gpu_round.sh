#!/usr/bin/env bash
# One GPU-box pass: GPU tests, the reference's own suite against the package,
# role-rotation A/B, per-sub-partition fp64 pipe balance of the probe kernel,
# the full bench. Usage: tools/gpu_round.sh TAG   (outputs gpurun_out/TAG_*)
set -u
TAG=${1:-rXX}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
GVP_PARITY_DUMP=$O timeout 1200 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 900 python tools/run_reference_suite.py > $O/${TAG}_refsuite.log 2>&1
echo "refsuite rc=$?" >> $O/${TAG}_refsuite.log
for ROT in 0 1; do
  GVP_PROBE_ROT=$ROT timeout 300 python bench.py --steps 10 --warmup 3 --no-c1 --no-c3 --no-cpu-baseline --no-converge \
    > $O/${TAG}_ab_rot$ROT.json 2> $O/${TAG}_ab_rot$ROT.err
done
for ROT in 0 1; do
  GVP_PROBE_ROT=$ROT timeout 600 ncu --kernel-name regex:probe_split --launch-skip 3 --launch-count 1 --clock-control none \
    --metrics gpu__time_duration.sum,smsp__pipe_fp64_cycles_active.max,smsp__pipe_fp64_cycles_active.avg,smsp__pipe_fp64_cycles_active.min,smsp__inst_executed.max,smsp__inst_executed.avg,smsp__inst_executed.min,smsp__cycles_active.avg,smsp__warps_active.avg.per_cycle_active \
    --csv python bench.py --steps 1 --warmup 3 --no-c1 --no-c3 --no-cpu-baseline --no-converge \
    > $O/${TAG}_ncu_balance_rot$ROT.csv 2> $O/${TAG}_ncu_balance_rot$ROT.err
done
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench rc=$?" >> $O/${TAG}_bench.err
