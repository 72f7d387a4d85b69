# round 2, GPU pass l: TMA bulk L2 prefetch D iterations past the ring (GV_RING_PF=D) on the DRAM-bound C5 and on C2
set -x
for v in def pf2 pf4 pf5; do
  if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
  timeout 900 python bench.py --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2l_c5_$v.json 2> gpurun_out/r2l_c5_$v.err; echo c5_$v=$?
  timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2l_c2_$v.json 2> gpurun_out/r2l_c2_$v.err; echo c2_$v=$?
done
export GV_LIB_PATH=paper_1903_00757_b200/libgv_pf4.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ring_kernel_math or hogwild_shapes" > gpurun_out/r2l_test_pf4.log 2>&1; echo test_pf4=$?
