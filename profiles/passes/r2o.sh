# round 2, GPU pass o: scatter stores through a per-bin destination address (no division per sample) — parity, C2 n = 4 / 16, C5 D = 8 bucketing launch list
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "bucketing or relabeled or device_blocks or processes_ordered" > gpurun_out/r2o_bucket.log 2>&1; echo bucket=$?
for pp in 4 16; do
  timeout 600 python bench.py --config C2 --parts-per-rank $pp --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2o_c2_n$pp.json 2> gpurun_out/r2o_c2_n$pp.err; echo c2n$pp=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bucket -c 60 --csv --log-file gpurun_out/r2o_c5_vr8_launches.csv python bench.py --vranks 8 --parts-per-rank 2 --pool 250000000 --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2o_launches.log 2>&1; echo launches=$?
