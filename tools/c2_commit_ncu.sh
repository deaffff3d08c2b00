O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:commit_kernel --launch-skip 10 --launch-count 1 -o /tmp/c2commit -f python tools/c2_breakdown.py > $O/r02bi_ncu.log 2>&1
ncu -i /tmp/c2commit.ncu-rep --page raw --csv > $O/r02bi_raw.csv 2>&1
ncu -i /tmp/c2commit.ncu-rep --page source --csv --print-source sass > $O/r02bi_sass.csv 2>&1
