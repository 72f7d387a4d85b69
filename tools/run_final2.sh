# full GPU suite, default bench, out-of-core bench, sanitizers
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_final2.log 2>&1; echo rc=$? >> gpurun_out/pytest_final2.log
python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err
python bench.py --host-partitions 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ooc4.json 2> gpurun_out/bench_ooc4.err
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_drive.py > gpurun_out/sanitize2_$tool.log 2>&1; echo rc=$? >> gpurun_out/sanitize2_$tool.log
done
