# round 2, GPU pass d: A/B of the ring kernel's delta paths (default red.global; GV_RING_TMA=3: vertex delta by TMA bulk reduce, LDGSTS loads; =4: same with TMA loads) — correctness on row-disjoint pools, then C2 and C5 rates
set -x
for v in def t3 t4; do
  if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ring_kernel_math or hogwild_shapes" > gpurun_out/r2d_test_$v.log 2>&1; echo test_$v=$?
  timeout 600 python bench.py --config C2 --steps 10 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2d_c2_$v.json 2> gpurun_out/r2d_c2_$v.err; echo c2_$v=$?
done
for v in def t3; do
  if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
  timeout 900 python bench.py --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2d_c5_$v.json 2> gpurun_out/r2d_c5_$v.err; echo c5_$v=$?
done
