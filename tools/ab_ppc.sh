# plans-per-CTA fill (auto lanes) across batch sizes, N = 1000
for B in 4096 3000 2048 1024 256 16 1; do
  timeout 300 python tools/sweep_batch.py one $B 1000 0 2>&1 | tail -1
done
