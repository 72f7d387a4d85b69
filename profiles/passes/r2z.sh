# round 2, GPU pass z: the D = 8 schedule of C5 on one GPU with vertex tiles (8 virtual ranks, n = 16: per-rank SGD / bucketing / tile sort / exchange), the n = 8 per-block kernel on C2 with tiles (hot-row contention), C4 with tiles
set -x
timeout 1500 python bench.py --vranks 8 --parts-per-rank 2 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline --no-extra --no-e2e > gpurun_out/r2z_c5_vr8.json 2> gpurun_out/r2z_c5_vr8.err; echo c5vr8=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2z_c5_vr8_launches.csv python bench.py --vranks 8 --parts-per-rank 2 --steps 1 --warmup 1 --no-cpu-baseline --no-pipeline --no-extra --no-e2e > gpurun_out/r2z_c5_vr8_launches.log 2>&1; echo vr8launches=$?
for b in 14 0; do
  GV_BLOCK_LAUNCH=1 timeout 600 python bench.py --config C2 --partitions 8 --vertex-tile $b --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-extra --no-e2e > gpurun_out/r2z_c2_n8_perblock_b$b.json 2> gpurun_out/r2z_c2_n8_perblock_b$b.err; echo c2n8_$b=$?
done
for b in 14 0; do
  timeout 900 python bench.py --config C4 --vertex-tile $b --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-extra > gpurun_out/r2z_c4_b$b.json 2> gpurun_out/r2z_c4_b$b.err; echo c4_$b=$?
done
