# A/B: register cap of the half-warp Hogwild kernel (min blocks per SM 2 / 3 / 4)
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_mb2.json 2>&1
for v in mb3 mb4; do GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>&1; done
