# hot-row contention check: C2-sized graphs with lower degree caps, n = 1 vs n = 8 on one GPU
for w in 3000 300; do for m in 1 8; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --wmax $w --parts-per-rank $m > gpurun_out/hot_w${w}_m$m.json 2> gpurun_out/hot_w${w}_m$m.err
done; done
