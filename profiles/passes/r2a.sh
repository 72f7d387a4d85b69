set -x
nproc; free -g; nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gputest.log 2>&1; echo gputest=$?
timeout 2400 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo bench=$?
tail -3 gpurun_out/r2a_gputest.log
