# round 2, GPU pass g: hot-row contention vs delta path — C2 n = 8 grid, one launch per block (a D = 8 GPU's kernel), default red.global vs TMA bulk reduce (t2: all rows, t3/t4: vertex row)
set -x
for v in def t2 t3 t4; do
  if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
  GV_BLOCK_LAUNCH=1 timeout 600 python bench.py --config C2 --parts-per-rank 8 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2g_c2n8_$v.json 2> gpurun_out/r2g_c2n8_$v.err; echo c2n8_$v=$?
  GV_BLOCK_LAUNCH=1 timeout 600 python bench.py --config C2 --parts-per-rank 4 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2g_c2n4_$v.json 2> gpurun_out/r2g_c2n4_$v.err; echo c2n4_$v=$?
done
unset GV_LIB_PATH
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2g_c2n1_def.json 2> gpurun_out/r2g_c2n1_def.err; echo c2n1=$?
