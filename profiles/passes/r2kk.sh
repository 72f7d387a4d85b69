# round 2, GPU pass kk: vertex rows kept in L2 with evict_last and no hint on context rows (GV_VTILE_HINT=2) vs no hints, C5 / C2 with tiles; smoke of the rebuilt library
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2kk_smoke.log 2>&1; echo smoke=$?
for h in 0 2; do
  GV_VTILE_HINT=$h timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e --no-extra > gpurun_out/r2kk_c5_h$h.json 2> gpurun_out/r2kk_c5_h$h.err; echo c5_$h=$?
  GV_VTILE_HINT=$h timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-pipeline --no-e2e --no-extra > gpurun_out/r2kk_c2_h$h.json 2> gpurun_out/r2kk_c2_h$h.err; echo c2_$h=$?
done
