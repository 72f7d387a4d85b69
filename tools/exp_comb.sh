# HISTORICAL: drives a hot-row combining / replica build that was withdrawn;
# its GV_COMB_* / GV_REP_* variables do nothing in the current library. Results: profiles/r01_hot_row_combining.json
# hot-row delta combining (on by default for n >= 4): GPU tests, then speed on C2 (n = 4, 8) and C4 (n = 32)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/comb_tests.log 2>&1; echo "rc=$?" >> gpurun_out/comb_tests.log
for cfg in "0 32 8" "16 16 8" "16 32 8" "16 64 8" "0 32 4" "16 32 4" "8 32 8"; do
  set -- $cfg
  GV_COMB_ROWS=$1 GV_COMB_FLUSHES=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $3 > gpurun_out/comb_H$1_F$2_m$3.json 2> gpurun_out/comb_H$1_F$2_m$3.err
done
for H in 0 16; do
  GV_COMB_ROWS=$H timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank 32 > gpurun_out/comb_c4_H$H.json 2> gpurun_out/comb_c4_H$H.err
done
