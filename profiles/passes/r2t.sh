# round 2, GPU pass t: the split kernel sources — smoke, full GPU suite, the default bench line, its launch list, 4 processes on one GPU (C2), and the reference arm
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2t_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2t_gputest.log 2>&1; echo gputest=$?
timeout 1800 python bench.py > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err; echo bench=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2t_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2t_launches.log 2>&1; echo launches=$?
GV_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 4 --config C2 --steps 3 --warmup 3 > gpurun_out/r2t_c2_4rank.json 2> gpurun_out/r2t_c2_4rank.err; echo c2_4rank=$?
timeout 1500 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2t_reference.json 2> gpurun_out/r2t_reference.err; echo reference=$?
tail -3 gpurun_out/r2t_gputest.log
