# round 2, GPU pass aa: tile-sort scratch sized by the digit in use — the vertex-tile tests (incl. CUDA-IPC processes, the sampler writing blocks), one 4e9-sample C5 pool with tiles (164 GB on the device)
set -x
timeout 1500 python -m pytest tests/test_gpu_vtile.py tests/test_gpu_multiprocess.py tests/test_gpu_parity.py -x -q -k "vtile or vertex_tile or processes or device_blocks" > gpurun_out/r2aa_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2aa_tests.log
timeout 1800 python bench.py --pool 4000000000 --steps 3 --warmup 1 --no-cpu-baseline --no-pipeline --no-extra > gpurun_out/r2aa_c5_pool4e9.json 2> gpurun_out/r2aa_c5_pool4e9.err; echo pool4e9=$?
tail -3 gpurun_out/r2aa_c5_pool4e9.err
