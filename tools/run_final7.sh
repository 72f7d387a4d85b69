# end-of-session capture: GPU suite, smoke, default bench line, its launch list, ncu --set full of the
# default SGD kernel (traffic), the 2-rank bench path on one GPU, and the reference (oracle) arm
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f7_pytest.log 2>&1; echo rc=$? >> gpurun_out/f7_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f7_smoke.log 2>&1; echo rc=$? >> gpurun_out/f7_smoke.log
timeout 600 python bench.py > gpurun_out/f7_bench.json 2> gpurun_out/f7_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f7_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/f7_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgd_ring -s 1 -c 1 -o gpurun_out/f7_prof python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-pipeline > gpurun_out/f7_ncu.log 2>&1
ncu -i gpurun_out/f7_prof.ncu-rep --page raw --csv > gpurun_out/f7_ring_raw.csv 2>&1
ncu -i gpurun_out/f7_prof.ncu-rep --page details --csv > gpurun_out/f7_ring_details.csv 2>&1
GV_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --pool 50000000 --no-cpu-baseline > gpurun_out/f7_bench_2rank.json 2> gpurun_out/f7_bench_2rank.err; echo rc=$? >> gpurun_out/f7_bench_2rank.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f7_reference.json 2> gpurun_out/f7_reference.err
