# round 2, GPU pass n: scatter reuses its multisplit masks (A/B vs pass m); ring depth P = 2 (12 warps/SM) vs P = 3 (8 warps/SM) on C2 and C5
set -x
timeout 600 python bench.py --config C2 --parts-per-rank 16 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2n_c2_n16.json 2> gpurun_out/r2n_c2_n16.err; echo c2n16=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bucket -c 60 --csv --log-file gpurun_out/r2n_c5_vr8_launches.csv python bench.py --vranks 8 --parts-per-rank 2 --pool 250000000 --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2n_launches.log 2>&1; echo launches=$?
for v in def p2; do
  if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
  timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2n_c2_$v.json 2> gpurun_out/r2n_c2_$v.err; echo c2_$v=$?
  timeout 900 python bench.py --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2n_c5_$v.json 2> gpurun_out/r2n_c5_$v.err; echo c5_$v=$?
done
unset GV_LIB_PATH
timeout 900 python -m pytest tests -m gpu -x -q -k "bucketing or relabeled" > gpurun_out/r2n_bucket.log 2>&1; echo bucket=$?
