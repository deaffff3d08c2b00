#!/usr/bin/env bash
# A/B of the probe kernel variants on C5 (GVP_PROBE=split|fused), short bench runs,
# then the parity tests under the last variant.
O=gpurun_out
SHORT="--steps 10 --warmup 3 --no-c1 --no-c3 --no-cpu-baseline --no-converge"
for V in ${*:-split fused}; do
  GVP_PROBE=$V timeout 300 python bench.py $SHORT > $O/ab_probe_$V.json 2> $O/ab_probe_$V.err
done
GVP_PROBE=$V GVP_PARITY_DUMP=$O timeout 900 python -m pytest tests/test_gpu_trace_parity.py tests/test_gpu_engine.py \
  tests/test_gpu_parity.py -q -s -p no:cacheprovider > $O/ab_probe_tests_$V.log 2>&1
