for v in pf0 pf8 pf16; do GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>&1; done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_pf4.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -s -k "hogwild_auc" > gpurun_out/auc5.log 2>&1; echo rc=$? >> gpurun_out/auc5.log
