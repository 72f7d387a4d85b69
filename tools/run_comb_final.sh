# HISTORICAL: drives a hot-row combining / replica build that was withdrawn;
# its GV_COMB_* / GV_REP_* variables do nothing in the current library. Results: profiles/r01_hot_row_combining.json
# combining on by default for n >= 4: full GPU suite, smoke, default bench (n = 1), n = 8 bench
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/cf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cf_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/cf_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/cf_smoke.log
timeout 400 python bench.py > gpurun_out/cf_bench.json 2> gpurun_out/cf_bench.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --parts-per-rank 8 > gpurun_out/cf_bench_n8.json 2> gpurun_out/cf_bench_n8.err
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --parts-per-rank 32 > gpurun_out/cf_bench_c4_n32.json 2> gpurun_out/cf_bench_c4_n32.err
