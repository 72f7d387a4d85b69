# bucketing CTAs per SM A/B (n = 4: single pass; n = 32: two-pass), C2 on one GPU
for c in 4 8 16; do for m in 4 32; do
  GV_BUCKET_CTAS=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $m > gpurun_out/abb_c${c}_m$m.json 2> gpurun_out/abb_c${c}_m$m.err
done; done
