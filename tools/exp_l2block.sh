# L2 blocking experiment: one-GPU n x n grid (parts-per-rank m) on C2 and C4
for m in 1 4 8 16 32; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $m > gpurun_out/l2b_c2_m$m.json 2> gpurun_out/l2b_c2_m$m.err
done
for m in 1 16 32 64; do
  timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $m > gpurun_out/l2b_c4_m$m.json 2> gpurun_out/l2b_c4_m$m.err
done
for m in 32; do
  timeout 600 python bench.py --config C4 --pool 800000000 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $m > gpurun_out/l2b_c4p8_m$m.json 2> gpurun_out/l2b_c4p8_m$m.err
done
