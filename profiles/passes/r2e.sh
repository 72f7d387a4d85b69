# round 2, GPU pass e: NEXT-1 sampler writing blocks directly — parity, then pipeline rates (blocks vs raw pools) on C2 at n = 1 and n = 4
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "device_blocks or device_pipeline or device_augmentation" > gpurun_out/r2e_blocks.log 2>&1; echo blocks=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2e_gputest.log 2>&1; echo gputest=$?
for pp in 1 4 16; do
  timeout 600 python bench.py --config C2 --parts-per-rank $pp --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-e2e > gpurun_out/r2e_c2_n${pp}_blocks.json 2> gpurun_out/r2e_c2_n${pp}_blocks.err; echo c2_${pp}_blocks=$?
  GV_AUG_BLOCKS=0 timeout 600 python bench.py --config C2 --parts-per-rank $pp --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-e2e > gpurun_out/r2e_c2_n${pp}_raw.json 2> gpurun_out/r2e_c2_n${pp}_raw.err; echo c2_${pp}_raw=$?
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2e_c2_n4_launches.csv python bench.py --config C2 --parts-per-rank 4 --steps 2 --warmup 1 --no-extra --no-cpu-baseline --no-e2e > gpurun_out/r2e_launches.log 2>&1; echo launches=$?
tail -3 gpurun_out/r2e_gputest.log
