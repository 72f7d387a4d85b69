# ncu of the default Hogwild kernel (ring) + GPU tests (full-size, pipeline) + bench line
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgd_ring -s 1 -c 1 -o gpurun_out/prof7 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full7.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "not hogwild_auc" > gpurun_out/pytest_gpu7.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu7.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench7.json 2> gpurun_out/bench7.err
