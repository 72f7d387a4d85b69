# Friendster-shaped (C5: 65.6M nodes, 1.8B edge draws, 2 x 33.6 GB embeddings) on ONE GPU
free -g > gpurun_out/c5_mem_before.txt
python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo rc=$? >> gpurun_out/bench_c5.err
