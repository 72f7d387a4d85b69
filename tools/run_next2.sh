# NEXT-2 ablations + shuffle-mode parity test
timeout 900 python -m pytest tests -m gpu -q -k "shuffle_modes or device_augmentation" > gpurun_out/pytest_next2.log 2>&1; echo rc=$? >> gpurun_out/pytest_next2.log
timeout 2400 python tools/ablations.py --out gpurun_out/next2_ablations.json > gpurun_out/next2_ablations.log 2>&1; echo rc=$? >> gpurun_out/next2_ablations.log
