# A/B: shared-memory ring depth P of the Hogwild kernel (default P=3), and the
# register half-warp kernel (GV_SGD_RING=0); C2 bench
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_p3.json 2>&1
GV_SGD_RING=0 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_reg.json 2>&1
for v in p2 p5 p8; do GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q -s -k "hogwild_auc" > gpurun_out/auc7.log 2>&1; echo rc=$? >> gpurun_out/auc7.log
