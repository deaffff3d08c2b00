O=gpurun_out
SHORT="--steps 10 --warmup 3 --no-c1 --no-c3 --no-cpu-baseline --no-converge"
timeout 300 python bench.py $SHORT > $O/r02m_lazy.json 2>&1
GVP_B200_LIB=paper_2411_03416_b200/var_nolazy/libgvp_b200.so timeout 300 python bench.py $SHORT > $O/r02m_nolazy.json 2>&1
timeout 300 python tools/c3_profile.py 10 > $O/r02m_c3_profile.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02m_c3_launches.csv python tools/c3_run.py --iters 5 > $O/r02m_c3_ncu.log 2>&1
