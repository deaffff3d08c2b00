set -x
for spec in "4096 2 base" "3552 2 base" "3552 4 base" "3552 4 pm3" "2960 4 pm3" "4096 4 pm3"; do
  set -- $spec
  lib=paper_2411_03416_b200/libgvp_b200.so; [ "$3" = pm3 ] && lib=variants/libgvp_pm3.so
  GVP_PROBE=split GVP_B200_LIB=$lib timeout 300 python tools/sweep_batch.py one $1 1000 $2 2>&1 | tail -1
done
