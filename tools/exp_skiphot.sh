# measurement-only: drop the deltas of the H hottest rows per partition (libgv_skiphot.so) at n = 8 and n = 1 on C2
export GV_LIB_PATH=paper_1903_00757_b200/libgv_skiphot.so
for H in 1 8 64 512; do for m in 1 8; do
  GV_HOT_ROWS=$H timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pipeline --parts-per-rank $m > gpurun_out/skh_H${H}_m$m.json 2> gpurun_out/skh_H${H}_m$m.err
done; done
