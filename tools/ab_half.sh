# A/B: full-warp (hw0) vs half-warp (default) Hogwild kernel, C2 bench + parity
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_hw1.json 2>&1
GV_LIB_PATH=paper_1903_00757_b200/libgv_hw0.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_hw0.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -s -k "hogwild_auc" > gpurun_out/auc6.log 2>&1; echo rc=$? >> gpurun_out/auc6.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_hogwild_kernel -s 1 -c 1 -o gpurun_out/prof6 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full6.log 2>&1
