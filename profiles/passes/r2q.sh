# round 2, GPU pass q: sampler-to-blocks placement v3 (destinations in shared memory, next walk prefetched) — parity and pipeline A/B (raw vs blocks) on C2 n = 1/4/16
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "device_blocks or device_pipeline" > gpurun_out/r2q_blocks.log 2>&1; echo blocks=$?
for pp in 1 4 16; do
  for ab in 0 1; do
    GV_AUG_BLOCKS=$ab timeout 600 python bench.py --config C2 --parts-per-rank $pp --steps 3 --warmup 3 --no-extra --no-cpu-baseline --no-e2e > gpurun_out/r2q_c2_n${pp}_ab$ab.json 2> gpurun_out/r2q_c2_n${pp}_ab$ab.err; echo c2_${pp}_$ab=$?
  done
done
GV_AUG_BLOCKS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:augment -c 40 --csv --log-file gpurun_out/r2q_c2_n4_aug_launches.csv python bench.py --config C2 --parts-per-rank 4 --steps 2 --warmup 1 --no-extra --no-cpu-baseline --no-e2e > gpurun_out/r2q_launches.log 2>&1; echo launches=$?
