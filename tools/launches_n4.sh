# per-kernel launch list for n = 4 partitions on one rank (bucketing cost)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n4.csv python bench.py --parts-per-rank 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/launches_n4.log 2>&1
