# C5 (Friendster-shaped) on one GPU with the n x n grid (L2 blocking), n = m
for m in 16 64; do
  timeout 1500 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $m > gpurun_out/c5p_m$m.json 2> gpurun_out/c5p_m$m.err
done
