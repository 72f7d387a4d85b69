# round 2, GPU pass c: relabelled pool ids — parity, default bench (C5), a 4e9-sample C5 pool on one GPU, C2 per-block n = 8 (hot-row contention baseline)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "relabeled" > gpurun_out/r2c_relabeled.log 2>&1; echo relabeled=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gputest.log 2>&1; echo gputest=$?
timeout 1800 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo bench=$?
GV_BLOCK_LAUNCH=1 timeout 600 python bench.py --config C2 --parts-per-rank 8 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2c_c2_n8_perblock.json 2> gpurun_out/r2c_c2_n8_perblock.err; echo c2n8=$?
timeout 1500 python bench.py --pool 4000000000 --steps 3 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline > gpurun_out/r2c_c5_pool4e9.json 2> gpurun_out/r2c_c5_pool4e9.err; echo pool4e9=$?
tail -3 gpurun_out/r2c_gputest.log
