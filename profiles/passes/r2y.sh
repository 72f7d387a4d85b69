# round 2, GPU pass y: the shipped build after R-VTILE + dynamic chunks — smoke, the whole GPU suite, the default bench line, its launch list, 4 processes on one GPU (C2, tiles after the fused exchange), compute-sanitizer over every kernel
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/r2y_smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2y_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/r2y_gputest.log
timeout 1800 python bench.py > gpurun_out/r2y_bench.json 2> gpurun_out/r2y_bench.err; echo bench=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2y_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2y_launches.log 2>&1; echo launches=$?
GV_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 4 --config C2 --steps 3 --warmup 3 > gpurun_out/r2y_c2_4rank.json 2> gpurun_out/r2y_c2_4rank.err; echo c2_4rank=$?
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/r2y_sanitize_$tool.log 2>&1; echo $tool=$?
done
