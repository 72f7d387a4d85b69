# round 2, GPU pass ff: ring-kernel geometry re-measured on tiled C5 / C2 pools (vertex rows from L2 change the latency mix): ring depth P = 2 / 3 (default) / 4, 16 lanes per sample
set -x
for v in def p2 p4 l16; do
  lib=paper_1903_00757_b200/libgv_$v.so; [ $v = def ] && lib=paper_1903_00757_b200/libgv.so
  GV_LIB_PATH=$lib timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e --no-extra > gpurun_out/r2ff_c5_$v.json 2> gpurun_out/r2ff_c5_$v.err; echo c5_$v=$?
  GV_LIB_PATH=$lib timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e --no-extra > gpurun_out/r2ff_c2_$v.json 2> gpurun_out/r2ff_c2_$v.err; echo c2_$v=$?
done
