# full GPU suite, default bench, 2-process bench with m = 2 on one GPU, sanitizers
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_final3.log 2>&1; echo rc=$? >> gpurun_out/pytest_final3.log
python bench.py > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err
GV_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --pool 50000000 --parts-per-rank 2 --no-cpu-baseline > gpurun_out/bench_mp_m2.json 2> gpurun_out/bench_mp_m2.err; echo rc=$? >> gpurun_out/bench_mp_m2.err
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize3_$tool.log 2>&1; echo rc=$? >> gpurun_out/sanitize3_$tool.log
done
