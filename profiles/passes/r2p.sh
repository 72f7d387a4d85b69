# round 2, GPU pass p: multi-process path with relabelled pools (tests) and the 2-process C5 bench on one GPU; full GPU suite
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_multiprocess.py -x -q > gpurun_out/r2p_mp.log 2>&1; echo mp=$?
GV_BENCH_DEVICE=0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2p_c5_2rank.json 2> gpurun_out/r2p_c5_2rank.err; echo c5_2rank=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/r2p_gputest.log
