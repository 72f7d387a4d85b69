# Friendster-small-shaped (C4) on one GPU: bench line + ncu of the SGD kernel
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo rc=$? >> gpurun_out/bench_c4.err
timeout 900 ncu --set full --clock-control none -k regex:sgd_ring -s 1 -c 1 -o gpurun_out/prof_c4 python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/ncu_c4.log 2>&1
