# round 2, GPU pass r (measurement only, wrong training): what a partial relief of hot-row contention could buy — drop all (skip1) or a quarter (skip2) of the deltas of the H hottest rows per partition, C2 n = 8, one launch per block
set -x
for v in skip1 skip2; do
  for H in 8 64; do
    GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so GV_HOT_ROWS=$H GV_BLOCK_LAUNCH=1 timeout 600 python bench.py --config C2 --parts-per-rank 8 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2r_c2n8_${v}_h$H.json 2> gpurun_out/r2r_c2n8_${v}_h$H.err; echo ${v}_$H=$?
  done
done
GV_BLOCK_LAUNCH=1 timeout 600 python bench.py --config C2 --parts-per-rank 8 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2r_c2n8_def.json 2> gpurun_out/r2r_c2n8_def.err; echo def=$?
