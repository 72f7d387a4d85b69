# HISTORICAL: drives a hot-row combining / replica build that was withdrawn;
# its GV_COMB_* / GV_REP_* variables do nothing in the current library. Results: profiles/r01_hot_row_combining.json
# combining option: quality test (n = 8, stalest setting), ring math on disjoint rows with it on, and n = 1 / 8 speed
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "hot_row_combining" > gpurun_out/comb3_quality.log 2>&1; echo "rc=$?" >> gpurun_out/comb3_quality.log
GV_COMB_ROWS=16 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "disjoint_rows or degenerate" > gpurun_out/comb3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/comb3_tests.log
for cfg in "0 8" "16 8" "0 4" "16 4" "0 1" "16 1"; do
  set -- $cfg
  GV_COMB_ROWS=$1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $2 > gpurun_out/comb3_H$1_m$2.json 2> gpurun_out/comb3_H$1_m$2.err
done
