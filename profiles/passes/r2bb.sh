# round 2, GPU pass bb: final validation of the shipped build — fresh build + smoke, the whole GPU suite, the default bench line, its launch list, the reference arm
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2bb_smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/r2bb_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2bb_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/r2bb_gputest.log
timeout 1800 python bench.py > gpurun_out/r2bb_bench.json 2> gpurun_out/r2bb_bench.err; echo bench=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2bb_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2bb_launches.log 2>&1; echo launches=$?
timeout 1500 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2bb_reference.json 2> gpurun_out/r2bb_reference.err; echo reference=$?
