set -u
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:step_kernel \
  --launch-skip 2 --launch-count 1 -o /tmp/c3step -f python tools/c3_run.py --iters 4 > $O/r02t_c3ncu.log 2>&1
ncu -i /tmp/c3step.ncu-rep --page raw --csv > $O/r02t_c3step_raw.csv 2>&1
ncu -i /tmp/c3step.ncu-rep --page source --csv --print-source sass > $O/r02t_c3step_sass.csv 2>&1
ncu -i /tmp/c3step.ncu-rep --page source --csv --print-source cuda > $O/r02t_c3step_cuda.csv 2>&1
ls -la $O/r02t_*
