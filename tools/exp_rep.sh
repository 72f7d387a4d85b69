# HISTORICAL: drives a hot-row combining / replica build that was withdrawn;
# its GV_COMB_* / GV_REP_* variables do nothing in the current library. Results: profiles/r01_hot_row_combining.json
# hot-row delta replicas: full-size quality first, parity tests, then speed on C2
#timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k quality_grid > gpurun_out/rep_quality.log 2>&1; echo "rc=$?" >> gpurun_out/rep_quality.log
#GV_REP_ROWS=16 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "disjoint_rows or degenerate or hogwild_auc or hogwild_shapes" > gpurun_out/rep_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rep_tests.log
for cfg in "x 8 4 8" "0 8 4 8" "x 8 1 8" "x 8 2 8" "x 8 8 8" "x 4 2 8" "x 8 4 4" "16 8 4 1"; do
  set -- $cfg
  if [ $1 = x ]; then unset GV_REP_ROWS; else export GV_REP_ROWS=$1; fi
  GV_REP_COPIES=$2 GV_REP_EVERY=$3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $4 > gpurun_out/rep_H$1_C$2_E$3_m$4.json 2> gpurun_out/rep_H$1_C$2_E$3_m$4.err
done
unset GV_REP_ROWS
