# round 2, GPU pass x: DRAM bytes of the tiled SGD kernel (C5, C2; single-pass ncu metrics, for profiles/sgd_traffic.json), ncu --set full of the tiled C5 SGD kernel and of the tile-sort scatter, A/B of the L2 hints with tiles (GV_VTILE_HINT)
set -x
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:sgd_ring -s 2 -c 1 --csv --log-file gpurun_out/r2x_c5_dram.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline --no-extra > gpurun_out/r2x_c5_dram.log 2>&1; echo c5dram=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:sgd_ring -s 2 -c 1 --csv --log-file gpurun_out/r2x_c2_dram.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline --no-extra > gpurun_out/r2x_c2_dram.log 2>&1; echo c2dram=$?
GV_VTILE_HINT=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-extra > gpurun_out/r2x_c5_hint.json 2> gpurun_out/r2x_c5_hint.err; echo c5hint=$?
GV_VTILE_HINT=1 timeout 900 python bench.py --vertex-tile 16 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-extra > gpurun_out/r2x_c5_hint16.json 2> gpurun_out/r2x_c5_hint16.err; echo c5hint16=$?
timeout 900 python bench.py --vertex-tile 16 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-extra > gpurun_out/r2x_c5_b16.json 2> gpurun_out/r2x_c5_b16.err; echo c5b16=$?
GV_VTILE_HINT=1 timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-extra > gpurun_out/r2x_c2_hint.json 2> gpurun_out/r2x_c2_hint.err; echo c2hint=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"sgd_ring|bucket_scatter_fast|bucket_hist" -s 3 -c 3 -o gpurun_out/r2x_c5_full python bench.py --pool 100000000 --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2x_c5_full.log 2>&1; echo c5full=$?
ncu -i gpurun_out/r2x_c5_full.ncu-rep --page details --csv > gpurun_out/r2x_c5_full_details.csv 2>&1
ncu -i gpurun_out/r2x_c5_full.ncu-rep --page raw --csv > gpurun_out/r2x_c5_full_raw.csv 2>&1
rm -f gpurun_out/*.ncu-rep
