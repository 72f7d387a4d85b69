# round 2, GPU pass i: partition lookup of relabelled ids by multiply-high (was a 64-bit division) — parity, then bucketing times (C2 n = 4 / 16 one GPU; C5 D = 8 schedule launch list)
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "relabeled or bucketing" > gpurun_out/r2i_relabeled.log 2>&1; echo relabeled=$?
for pp in 4 16; do
  timeout 600 python bench.py --config C2 --parts-per-rank $pp --vranks 1 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2i_c2_n${pp}.json 2> gpurun_out/r2i_c2_n${pp}.err; echo c2_$pp=$?
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2i_c5_vr8_launches.csv python bench.py --vranks 8 --parts-per-rank 2 --pool 250000000 --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2i_launches.log 2>&1; echo launches=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/r2i_gputest.log
