# NEXT-1 device augmentation: parity tests + bench with the pipeline detail
timeout 900 python -m pytest tests -m gpu -x -q -k "device_augmentation or device_pipeline or collaboration" > gpurun_out/pytest_next1.log 2>&1; echo rc=$? >> gpurun_out/pytest_next1.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_next1.json 2> gpurun_out/bench_next1.err
