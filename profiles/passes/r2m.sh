# round 2, GPU pass m: histogram without warp aggregation above 32 bins (issue-bound kernel) — A/B on C2 n = 16 and the C5 D = 8 launch list; smoke + full GPU suite
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2m_smoke.log 2>&1; echo smoke=$?
for v in def hagg; do
  if [ $v = def ]; then unset GV_LIB_PATH; else export GV_LIB_PATH=paper_1903_00757_b200/libgv_$v.so; fi
  timeout 600 python bench.py --config C2 --parts-per-rank 16 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2m_c2_n16_$v.json 2> gpurun_out/r2m_c2_n16_$v.err; echo c2_$v=$?
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bucket -c 60 --csv --log-file gpurun_out/r2m_c5_vr8_launches_$v.csv python bench.py --vranks 8 --parts-per-rank 2 --pool 250000000 --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-pipeline --no-e2e > gpurun_out/r2m_launches_$v.log 2>&1; echo launches_$v=$?
done
unset GV_LIB_PATH
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2m_gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/r2m_gputest.log
