# A/B: L2 retention hints (hot rows evict_last, cold rows evict_first) in the ring kernel
GV_HOT_ROWS=0 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_hot0.json 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_hotdef.json 2>&1
for h in 30000 150000 300000; do GV_HOT_ROWS=$h python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_hot$h.json 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_ring -s 1 -c 1 -o gpurun_out/prof8 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full8.log 2>&1
