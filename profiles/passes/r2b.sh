# round 2, GPU pass b: engine split verification, 2-process C5 on one GPU, ncu launch list + C5 DRAM bytes
set -x
df -h /dev/shm /tmp | cat
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_gputest.log 2>&1; echo gputest=$?
GV_BENCH_DEVICE=0 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config C5 --steps 3 --warmup 3 > gpurun_out/r2b_c5_2rank.json 2> gpurun_out/r2b_c5_2rank.err; echo c5_2rank=$?
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sgd_ring -s 2 -c 1 --csv --log-file gpurun_out/r2b_c5_dram.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline --no-extra > gpurun_out/r2b_c5_dram.log 2>&1; echo c5dram=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2b_launches.log 2>&1; echo launches=$?
tail -3 gpurun_out/r2b_gputest.log
