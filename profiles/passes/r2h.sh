# round 2, GPU pass h: the D = 8 schedule of C5 on one GPU (8 virtual ranks, m = 2, n = 16): per-rank bucketing / exchange / exposed rotation at full size
set -x
timeout 1500 python bench.py --vranks 8 --parts-per-rank 2 --pool 250000000 --steps 3 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline > gpurun_out/r2h_c5_vr8.json 2> gpurun_out/r2h_c5_vr8.err; echo c5vr8=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2h_c5_vr8_launches.csv python bench.py --vranks 8 --parts-per-rank 2 --pool 250000000 --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2h_launches.log 2>&1; echo launches=$?
