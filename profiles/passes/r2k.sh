# round 2, GPU pass k: ncu --set full of the bucketing kernels (C2, n = 16, single pass) and of the block-SGD kernel on C5 (1e8-sample pool)
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bucket_hist_kernel|bucket_scatter_fast" -s 2 -c 2 -o gpurun_out/r2k_bucket python bench.py --config C2 --parts-per-rank 16 --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2k_bucket.log 2>&1; echo bucket=$?
ncu -i gpurun_out/r2k_bucket.ncu-rep --page details --csv > gpurun_out/r2k_bucket_details.csv 2>&1
ncu -i gpurun_out/r2k_bucket.ncu-rep --page raw --csv > gpurun_out/r2k_bucket_raw.csv 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sgd_ring -s 1 -c 1 -o gpurun_out/r2k_c5_sgd python bench.py --pool 100000000 --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2k_c5_sgd.log 2>&1; echo c5sgd=$?
ncu -i gpurun_out/r2k_c5_sgd.ncu-rep --page details --csv > gpurun_out/r2k_c5_sgd_details.csv 2>&1
ncu -i gpurun_out/r2k_c5_sgd.ncu-rep --page raw --csv > gpurun_out/r2k_c5_sgd_raw.csv 2>&1
rm -f gpurun_out/*.ncu-rep
