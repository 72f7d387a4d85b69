# HISTORICAL: drives a hot-row combining / replica build that was withdrawn;
# its GV_COMB_* / GV_REP_* variables do nothing in the current library. Results: profiles/r01_hot_row_combining.json
# combining chosen from partition hotness: GPU suite, smoke, benches (C2 n = 1 / 4 / 8, C4 n = 32)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/cp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cp_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/cp_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/cp_smoke.log
timeout 400 python bench.py > gpurun_out/cp_bench.json 2> gpurun_out/cp_bench.err
for m in 4 8; do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --parts-per-rank $m > gpurun_out/cp_bench_n$m.json 2> gpurun_out/cp_bench_n$m.err
done
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --parts-per-rank 32 > gpurun_out/cp_bench_c4_n32.json 2> gpurun_out/cp_bench_c4_n32.err
