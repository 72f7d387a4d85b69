# HISTORICAL: drives a hot-row combining / replica build that was withdrawn;
# its GV_COMB_* / GV_REP_* variables do nothing in the current library. Results: profiles/r01_hot_row_combining.json
# combining: fixed flush iterations (GV_COMB_ITERS) vs per-launch count, C2 n = 8, repeated
for rep in 1 2; do
for cfg in "0 0" "16 256" "16 165" "16 64" "16 1024"; do  # GV_COMB_ITERS was a temporary A/B knob, now GV_COMB_FLUSH
  set -- $cfg
  GV_COMB_ROWS=$1 GV_COMB_ITERS=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank 8 > gpurun_out/comb2_H$1_I$2_r$rep.json 2> gpurun_out/comb2_H$1_I$2_r$rep.err
done; done
