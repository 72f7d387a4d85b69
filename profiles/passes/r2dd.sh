# round 2, GPU pass dd (measurement only, wrong training): hot-row contention with the dynamic chunk schedule — drop all (skip1), a quarter (skip2) or three quarters (skip3: each hot address sees the 1/4 load a 4-way sharded row would) of the deltas of the H hottest rows per partition; C2 n = 8, one launch per block, pool order
set -x
GV_BLOCK_LAUNCH=1 timeout 600 python bench.py --config C2 --partitions 8 --vertex-tile 0 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2dd_c2n8_def.json 2> gpurun_out/r2dd_c2n8_def.err; echo def=$?
for v in skip1 skip2 skip3; do
  for H in 8 64; do
    GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so GV_HOT_ROWS=$H GV_BLOCK_LAUNCH=1 timeout 600 python bench.py --config C2 --partitions 8 --vertex-tile 0 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2dd_c2n8_${v}_h$H.json 2> gpurun_out/r2dd_c2n8_${v}_h$H.err; echo ${v}_$H=$?
  done
done
