#!/usr/bin/env bash
# One GPU-box pass. Usage: tools/gpu_round.sh TAG [stages...]
# stages: tests refsuite c4 ncuprobe ncufactor bench abrot (default: tests refsuite bench)
set -u
TAG=${1:-rXX}; shift || true
STAGES=${*:-tests refsuite bench}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
SHORT="--steps 2 --warmup 3 --no-c1 --no-c3 --no-cpu-baseline --no-converge"
for st in $STAGES; do
  case $st in
    tests)
      GVP_PARITY_DUMP=$O timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > $O/${TAG}_pytest_gpu.log 2>&1
      echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log ;;
    refsuite)
      timeout 900 python tools/run_reference_suite.py > $O/${TAG}_refsuite.log 2>&1
      echo "refsuite rc=$?" >> $O/${TAG}_refsuite.log ;;
    c4)
      timeout 900 python tools/c4_n300.py > $O/${TAG}_c4_n300.jsonl 2> $O/${TAG}_c4_n300.err ;;
    ncuprobe)
      timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:probe_split \
        --launch-skip 3 --launch-count 1 -o $O/${TAG}_probe -f python bench.py $SHORT > $O/${TAG}_ncuprobe.log 2>&1 ;;
    ncucommit)
      timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:commit_kernel \
        --launch-skip 3 --launch-count 1 -o $O/${TAG}_commit -f python bench.py $SHORT > $O/${TAG}_ncucommit.log 2>&1 ;;
    ncufactor)
      timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:factor_grads \
        --launch-skip 5 --launch-count 1 -o $O/${TAG}_factor -f python bench.py $SHORT > $O/${TAG}_ncufactor.log 2>&1 ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file $O/${TAG}_launches.csv python bench.py $SHORT > $O/${TAG}_launches.log 2>&1 ;;
    abrot)
      for ROT in 0 1; do
        GVP_PROBE_ROT=$ROT timeout 300 python bench.py --steps 10 $(echo $SHORT | cut -d' ' -f3-) > $O/${TAG}_ab_rot$ROT.json 2>&1
      done ;;
    bench)
      timeout 1200 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
      echo "bench rc=$?" >> $O/${TAG}_bench.err ;;
  esac
done
