# full GPU suite + default bench line + ncu of the default Hogwild kernel (C2)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_final1.log 2>&1; echo rc=$? >> gpurun_out/pytest_final1.log
python bench.py > gpurun_out/bench_final1.json 2> gpurun_out/bench_final1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_ring -s 1 -c 1 -o gpurun_out/prof_final1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/ncu_final1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/ncu_launch_final1.log 2>&1
