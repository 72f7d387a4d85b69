# round 2, GPU pass j: single-pass bucketing up to 256 bins (n <= 16) vs the two-pass split at 128 bins — parity, C2 n = 16 rate, C5 D = 8 launch list
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "relabeled or bucketing or device_blocks or ordered_mode" > gpurun_out/r2j_bucket.log 2>&1; echo bucket=$?
for mb in 256 128; do
  GV_BUCKET_ONE_PASS_BINS=$mb timeout 600 python bench.py --config C2 --parts-per-rank 16 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2j_c2_n16_$mb.json 2> gpurun_out/r2j_c2_n16_$mb.err; echo c2_$mb=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2j_c5_vr8_launches.csv python bench.py --vranks 8 --parts-per-rank 2 --pool 250000000 --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2j_launches.log 2>&1; echo launches=$?
