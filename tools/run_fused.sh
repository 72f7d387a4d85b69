# fused scatter+exchange: virtual-rank and multi-process parity, bench with vranks and 2 processes
timeout 1500 python -m pytest tests -m gpu -q -x -k "vr or multiprocess or bucketing or negative or ordered or hogwild_auc or many_partitions or replay" > gpurun_out/pytest_fused.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused.log
python bench.py --vranks 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_fused_vr4.json 2> gpurun_out/bench_fused_vr4.err
GV_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --pool 50000000 --no-cpu-baseline > gpurun_out/bench_fused_mp2.json 2> gpurun_out/bench_fused_mp2.err; echo rc=$? >> gpurun_out/bench_fused_mp2.err
