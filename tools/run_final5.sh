# full GPU suite, default bench, launch list of the bench command, sanitizers, 2-process bench
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_final5.log 2>&1; echo rc=$? >> gpurun_out/pytest_final5.log
python bench.py > gpurun_out/bench_final5.json 2> gpurun_out/bench_final5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/ncu_launch_final5.log 2>&1
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize5_$tool.log 2>&1; echo rc=$? >> gpurun_out/sanitize5_$tool.log
done
GV_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --pool 50000000 --no-cpu-baseline > gpurun_out/bench_mp5.json 2> gpurun_out/bench_mp5.err; echo rc=$? >> gpurun_out/bench_mp5.err
