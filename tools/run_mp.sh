# multi-process (CUDA IPC) tests on one GPU + the full GPU suite
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -x -q > gpurun_out/pytest_mp.log 2>&1; echo rc=$? >> gpurun_out/pytest_mp.log
timeout 1500 python -m pytest tests -m gpu -x -q -k "not multiprocess" > gpurun_out/pytest_all.log 2>&1; echo rc=$? >> gpurun_out/pytest_all.log
