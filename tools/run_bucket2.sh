# faster bucketing (warp-aggregated histogram, register/shared-memory sorted scatter): parity + launch list
timeout 1500 python -m pytest tests -m gpu -q -x -k "bucketing or vr or multiprocess or ordered or negative or fullsize or out_of_core" > gpurun_out/pytest_bucket2.log 2>&1; echo rc=$? >> gpurun_out/pytest_bucket2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n4b.csv python bench.py --parts-per-rank 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/launches_n4b.log 2>&1
python bench.py --vranks 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_b2_vr4.json 2> gpurun_out/bench_b2_vr4.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/bench_b2_n1.json 2> gpurun_out/bench_b2_n1.err
