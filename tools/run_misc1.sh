bash tools/run_sanitize.sh
timeout 900 python -m pytest tests -m gpu -x -q -s -k "hogwild_auc" > gpurun_out/auc9.log 2>&1; echo rc=$? >> gpurun_out/auc9.log
python bench.py --vranks 8 --pool 25000000 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/bench_vr8.json 2> gpurun_out/bench_vr8.err
python bench.py --vranks 4 --pool 50000000 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/bench_vr4.json 2> gpurun_out/bench_vr4.err
