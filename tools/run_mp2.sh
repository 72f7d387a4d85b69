# multi-process Hogwild test + the torchrun bench path with 2 ranks sharing GPU 0
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -x -q > gpurun_out/pytest_mp2.log 2>&1; echo rc=$? >> gpurun_out/pytest_mp2.log
GV_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --pool 50000000 --no-cpu-baseline > gpurun_out/bench_mp2.json 2> gpurun_out/bench_mp2.err; echo rc=$? >> gpurun_out/bench_mp2.err
