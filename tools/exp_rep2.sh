# HISTORICAL: drives a hot-row combining / replica build that was withdrawn;
# its GV_COMB_* / GV_REP_* variables do nothing in the current library. Results: profiles/r01_hot_row_combining.json
# hot-row delta replicas: merge period sweep at n = 8 (C2), then full-size quality at the longest period
for E in 16 32 64; do
  GV_REP_EVERY=$E timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank 8 > gpurun_out/rep2_E$E.json 2> gpurun_out/rep2_E$E.err
done
GV_REP_EVERY=32 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s -k quality_grid > gpurun_out/rep2_quality.log 2>&1; echo "rc=$?" >> gpurun_out/rep2_quality.log
